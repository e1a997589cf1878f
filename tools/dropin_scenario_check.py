import sys, math, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import pyorc
from paper_1705_00614_b200.types import *
nx, ny = 96, 80
T = Terrain(nx, ny, 25.0, 0.0, 0.0, np.zeros(nx*ny))
for j in range(ny):
    for i in range(nx):
        T.b[i + j*nx] = 1e-3 * T.xc(i) + 0.7 * math.cos(0.11*i) * math.sin(0.07*j)
P = PhysicalParams(nu=0.5, omega_z=latitude_to_omega_z(48.7))
O = StepperOptions(boundaries=BoundaryConfig(EdgeKind.Reflective, EdgeKind.Open, EdgeKind.Reflective, EdgeKind.Reflective))
S = FlowState.dry(T)
for j in range(ny):
    for i in range(nx//3):
        S.H[i+j*nx] = max(0.0, 2.5 - T.b[i+j*nx])
src = [SourceSpec(SourceKind.Discharge, "drain", CellRect(70,30,72,33), [HydrographSample(0,-5.0), HydrographSample(50,-20.0)]),
       SourceSpec(SourceKind.Rain, "rain", CellRect(10,50,40,70), [], 2e-5)]
from paper_1705_00614_b200 import CsphTvdStepper
S2 = S.copy()
o = pyorc.OracleStepper(T, P, TimestepControl(), O)
g = CsphTvdStepper(T, P, TimestepControl(), O)
for x in (o, g):
    x.set_wind(WindForcing.constant(4.0,-1.0)); x.set_sources(src)
for n in range(40):
    a = o.step(S)
    try:
        b = g.step(S2)
    except Exception as e:
        print("gpu failed at step", n, e); break
    if a.tau != b.tau or not np.array_equal(S.H, S2.H):
        print("diverged at step", n, a.tau, b.tau, np.abs(S.H-S2.H).max()); break
else:
    print("gpu == oracle", S.t, S2.t)
