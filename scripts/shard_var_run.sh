#!/bin/bash
# Run scripts/shard_diag.py for every variants/clk_*.so (schedule / launch experiments at the
# kv-head shard shapes); one JSON line per (variant, config, P).
for so in variants/clk_*.so; do
  echo "== $(basename $so)"
  TA_LIBRARY=$PWD/$so timeout 300 python scripts/shard_diag.py "$@" 2>&1 | grep '^{'
done
