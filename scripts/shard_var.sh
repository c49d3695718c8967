for v in a_cur b_div2 c_div1; do echo "== $v"; TA_LIBRARY=$PWD/variants/clk_$v.so timeout 300 python scripts/shard_diag.py C2 C3 | grep -E '"P": (1|8)' | cut -c1-200; done
