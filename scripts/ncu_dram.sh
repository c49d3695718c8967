#!/bin/bash
# DRAM bytes of one C3 triangle attn_kernel launch for each given library build:
#   bash scripts/ncu_dram.sh variants/clk_base.so variants/clk_lqfirst.so ...
mkdir -p gpurun_out
for so in "$@"; do
  TA_LIBRARY=$PWD/$so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:attn_kernel -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dense --no-e2e --no-points 2>/dev/null \
    | grep -E '"dram__|"gpu__time' | awk -F'","' -v so=$so '{print so, $(NF-2), $(NF-1), $NF}'
done
