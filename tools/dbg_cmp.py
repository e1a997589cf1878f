import numpy as np, sys
a = np.load(sys.argv[1]); b = np.load(sys.argv[2])
for k in [1, 2, 3, 4, 5, 8, 16, 32, 64]:
    d = [int((a[f"{f}{k}"].view(np.uint64) != b[f"{f}{k}"].view(np.uint64)).sum()) for f in "HUV"]
    idx = np.flatnonzero(a[f"H{k}"].view(np.uint64) != b[f"H{k}"].view(np.uint64))[:5]
    print(k, d, [(int(i) % 128, int(i) // 128) for i in idx], a.get(f"redo{k}"), b.get(f"redo{k}"))
