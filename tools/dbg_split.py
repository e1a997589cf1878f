import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
mode = sys.argv[1]; out = sys.argv[2]
sc = S.lake_at_rest(128)
st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
s = sc.state.copy()
st.upload(s)
res = {}
done = 0
for k in [1, 2, 3, 4, 5, 8, 16, 32, 64]:
    n = k - done
    if mode == "run":
        st.run(n)
    else:
        for _ in range(n):
            st.step_resident()
    done = k
    st.download(s)
    res[f"H{k}"] = s.H.copy(); res[f"U{k}"] = s.HUx.copy(); res[f"V{k}"] = s.HUy.copy()
    try:
        res[f"redo{k}"] = np.array(st.redo_counts())
    except Exception:
        pass
np.savez(out, **res)
print("ok", mode)
