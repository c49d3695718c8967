#!/bin/bash
# Development loop on the GPU box: parity tests against a watchdog build (deadlocks trap
# instead of hanging), the variant timings, and the TA_TRACE timeline of CTA 0.
mkdir -p gpurun_out
if [ -f dbg/lib_wd.so ]; then
  TA_LIBRARY=$PWD/dbg/lib_wd.so timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pt_wd.log 2>&1
  rc=$?
  echo "pytest rc=$rc"; tail -3 gpurun_out/pt_wd.log
  if [ $rc != 0 ]; then exit 1; fi
fi
timeout 300 python scripts/variant_bench.py "$@" 2>&1 | tail -12
if [ "${TRACE:-1}" = "1" ]; then
  timeout 120 python scripts/trace_timeline.py C3 > gpurun_out/trace_c3.txt 2>&1
  grep -v "^ *-\?[0-9]* [A-Z][A-Z]\." gpurun_out/trace_c3.txt | tail -16
fi
