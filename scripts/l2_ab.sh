for r in 1 2 3; do
for m in flush inputs; do
python bench.py --no-cpu-baseline --no-e2e --no-dense --steps 100 --l2 $m | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$m', round(d['ms_per_layer'],4), d['clocks']['sm_mhz'], round(d['kernel_ms']['attn'],4))"
done; done
