import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1705_00614_b200 import scenarios as S
from test_gpu_nest import _gpu
from paper_1705_00614_b200.nesting import coupled_step
for r, win in [(3, (18, 21, 15, 11)), (4, (20, 20, 16, 16))]:
    ns = S.nested_floodplain(64, 50.0, win, r, 2)
    coarse, nest = _gpu(ns)
    for k in range(6):
        gi = coupled_step(coarse, [nest])
        print(r, k, gi.tau, gi.substeps_total, gi.fine_tau_min, gi.reflux_clamp_volume, flush=True)
