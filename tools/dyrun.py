"""Run a few dycore steps (512x512x80 f64) eagerly -- for ncu captures."""
import sys
sys.path.insert(0, '.')
import paper_2311_08322_b200 as b200
from paper_2311_08322_b200 import native, workloads
dom = (512, 512, 80)
st = b200.compile_stencil(workloads.source("dycore"), "dycore")
arr = workloads.dycore_arrays(dom, 0)
A, B = b200.from_array(arr["u"], (2, 2, 0)), b200.from_array(arr["u"], (2, 2, 0))
coef = {n: b200.from_array(arr[n]) for n in "abc"}
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    src, dst = (A, B) if s % 2 == 0 else (B, A)
    st(u_in=src, u_out=dst, **coef, **workloads.DYCORE_SCALARS)
native.synchronize()
print("ok", st.build_info["plan"])
