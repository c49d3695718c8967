#!/bin/bash
# memcheck + synccheck + racecheck on C1 triangle/dense and Llama N = 4097 (final build)
set -u
TAG=${1:-r02b}
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for case in 1 0 4; do
    log=gpurun_out/sanitize_${TAG}_${tool}_case${case}.log
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    CASE=$case timeout 900 compute-sanitizer --tool $tool $extra python scripts/debug_small.py > $log 2>&1
    echo "$tool case$case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1) $(grep -E '^n=' $log | tail -1)"
    if [ $tool = racecheck ]; then grep -E "at ta::" $log | sed 's/Thread ([0-9,]*)//; s/+0x[0-9a-f]*//' | sort | uniq -c | head -6; fi
  done
done
