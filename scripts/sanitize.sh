#!/bin/bash
# compute-sanitizer tiers (SURVEY 4 tier 7 / 5): memcheck, racecheck, synccheck, initcheck on
# C1 (triangle + dense) and the Llama shape at N = 4097 (triangle), each run through the C ABI
# (scripts/debug_small.py also checks the result against the oracle).
# Usage (GPU box): bash scripts/sanitize.sh TAG   -> gpurun_out/sanitize_TAG_<tool>_<case>.log
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for case in 1 0 4; do
    log=gpurun_out/sanitize_${TAG}_${tool}_case${case}.log
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    CASE=$case timeout 900 compute-sanitizer --tool $tool $extra python scripts/debug_small.py > $log 2>&1
    echo "$tool case$case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1) $(grep -E '^n=' $log | tail -1)"
  done
done
