#!/bin/bash
# Round profile capture (run on the GPU box via gpurun; outputs in gpurun_out/).
#   1. launch list of a short bench run (per-launch device time, serialized, cold)
#   2. one full ncu capture of each hot kernel: vadv TMEM column kernel,
#      hdiff f64/f32 fused PARALLEL kernel, the fused dycore column kernel
set -x
R=${1:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 --no-graph > gpurun_out/launches_bench_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k0_column_tmem -s 5 -c 1 -o gpurun_out/vadv_$R \
    python bench.py --steps 10 --warmup 5 --no-extra --no-cpu-baseline --e2e-steps 1 --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pfused -s 6 -c 1 -o gpurun_out/hdiff64_$R \
    python tools/ksweep.py hdiff f64 256x256x80 '{}' --eager=10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pfused -s 6 -c 1 -o gpurun_out/hdiff32_$R \
    python tools/ksweep.py hdiff f32 256x256x80 '{}' --eager=10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_column_tmem -s 3 -c 1 -o gpurun_out/dycore_$R \
    python tools/ksweep.py dycore f64 512x512x80 '{}' > /dev/null 2>&1
# DRAM traffic with the write-back included (range replay over [launch, read-only L2 eviction])
for w in vadv hdiff hdiff32 dycore; do
  ncu --replay-mode range --cache-control all --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file gpurun_out/traffic_$w.csv python tools/ncu_traffic.py $w > gpurun_out/traffic_$w.json 2>&1
done
ls -la gpurun_out
