#!/bin/bash
# Round-2 final evidence on one B200 (run via gpurun; outputs in gpurun_out/):
# GPU test suite, smoke, the bench line (both arms), a 2-rank shared-GPU bench
# (peer / fused transports), the launch list and the ncu captures.
set -x
R=${1:-r2f}
python -m pytest tests -m gpu -q > gpurun_out/gputest_$R.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.txt 2>&1
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
python bench.py --impl reference > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
GTS_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 200 --warmup 5 \
    > gpurun_out/bench_n2_shared_$R.json 2> gpurun_out/bench_n2_shared_$R.err
bash profiles/capture.sh $R
