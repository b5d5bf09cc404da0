"""Per-call cost of the reference-facing API (CompiledStencil.__call__) with
device-resident storages: wall clock per call (host overhead + launch +
kernel + the run() contract's stream synchronisation), vs the kernel alone."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import native, workloads  # noqa: E402

for kernel, dom in (("vadv", (256, 256, 80)), ("vadv", (8, 8, 8)), ("hdiff", (256, 256, 80)), ("hdiff", (8, 8, 8))):
    st = b200.compile_stencil(workloads.source(kernel), kernel)
    args = workloads.make_args(kernel, dom)
    for _ in range(20):
        st(**args)
    for validate in (True, False):
        n = 300
        t0 = time.perf_counter()
        for _ in range(n):
            rep = st(**args, validate=validate)
        dt = (time.perf_counter() - t0) / n
        print(f"{kernel} {dom} validate={validate}: {dt * 1e6:.1f} us/call wall; "
              f"report total {rep.total_ns / 1e3:.1f} us kernel {rep.kernel_ns / 1e3:.1f} us", flush=True)
