#!/bin/bash
# Round-end style GPU session: tests, smoke, bench (+sweep), reference arm, ncu launch list + full capture,
# compute-sanitizer memcheck on a small case.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 600 python -m pytest tests -m gpu -q --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_${TAG}.log)"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --sweep > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-points > gpurun_out/ncu_launch_bench_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 \
  -o gpurun_out/prof_attn_${TAG} -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dense --no-e2e --no-points > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
CASE=3 timeout 600 compute-sanitizer --tool memcheck --leak-check no python scripts/debug_small.py > gpurun_out/memcheck_${TAG}.log 2>&1; echo "memcheck rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/memcheck_${TAG}.log | tail -1)"
timeout 900 python scripts/ttft_synth.py > gpurun_out/ttft_${TAG}.json 2> gpurun_out/ttft_${TAG}.err; echo "ttft rc=$?"
