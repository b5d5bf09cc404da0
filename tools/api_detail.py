import sys, time
sys.path.insert(0, '/root/repo')
import paper_2311_08322_b200 as b200
from paper_2311_08322_b200 import native, workloads
for kernel, dom in (("vadv", (256, 256, 80)), ("vadv", (8, 8, 8))):
    st = b200.compile_stencil(workloads.source(kernel), kernel)
    args = workloads.make_args(kernel, dom)
    mod = st.build_info["module"]
    s = native.default_stream()
    fields = {k: v for k, v in args.items() if hasattr(v, "base_address")}
    go = mod.launcher(dom, fields, {}, s)
    for _ in range(10): go()
    native.synchronize(s)
    n = 200
    t0 = time.perf_counter()
    for _ in range(n): go()
    t1 = time.perf_counter()
    native.synchronize(s)
    t2 = time.perf_counter()
    print(kernel, dom, f"enqueue {1e6*(t1-t0)/n:.1f} us/launch, enqueue+drain {1e6*(t2-t0)/n:.1f} us/launch")
    t0 = time.perf_counter()
    for _ in range(n):
        go(); native.synchronize(s)
    t1 = time.perf_counter()
    print(kernel, dom, f"launch+sync {1e6*(t1-t0)/n:.1f} us")
    e0, e1 = native.Event(), native.Event()
    ts = []
    for _ in range(50):
        e0.record(s); go(); e1.record(s); native.synchronize(s); ts.append(e0.elapsed_ms(e1)*1e3)
    ts.sort(); print(kernel, dom, f"event-timed single launch median {ts[25]:.1f} us")
