import sys, os
sys.path.insert(0, os.getcwd())
from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
sc = S.floodplain(256, 50.0)
st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
st.set_wind(sc.wind); st.set_sources(sc.sources)
s = sc.state.copy(); st.upload(s)
for k in range(3):
    st.step_resident(); print("step", k, flush=True)
print("ok")
