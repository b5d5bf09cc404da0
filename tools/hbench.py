import sys
sys.path.insert(0, '.')
import paper_2311_08322_b200 as b200
from paper_2311_08322_b200 import workloads, native
dom = (256, 256, 80)
for dt in sys.argv[1:] or ["f64"]:
    st = b200.compile_stencil(workloads.source("hdiff", dt), "hdiff")
    sets = [workloads.make_args("hdiff", dom, dt, seed=s) for s in range(3)]
    stream = native.default_stream()
    gos = [st.build_info["module"].launcher(dom, {k: v for k, v in a.items() if hasattr(v, "base_address")}, {"coeff": 0.05}, stream) for a in sets]
    for i in range(6): gos[i % 3]()
    native.synchronize(stream)
    e0, e1 = native.Event(), native.Event()
    e0.record(stream)
    for i in range(60): gos[i % 3]()
    e1.record(stream); native.synchronize(stream)
    us = e0.elapsed_ms(e1) / 60 * 1000
    alg = workloads.algorithmic_bytes("hdiff", dom, dt)
    print(dt, st.build_info["plan"], f"{us:.2f} us", f"{alg/us/1e3:.0f} GB/s")
