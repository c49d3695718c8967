#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list, ncu --set full of the attention kernel.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_${TAG}.log)"
if [ "${SKIP_BENCH:-0}" != "1" ]; then
bash scripts/gpu_bench_profile.sh ${TAG}
fi
