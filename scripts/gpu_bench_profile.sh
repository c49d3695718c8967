#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list, one ncu --set full capture.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
nproc > gpurun_out/nproc.txt
timeout 900 python bench.py --sweep > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench_${TAG}.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 \
  -o gpurun_out/prof_attn_${TAG} -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
