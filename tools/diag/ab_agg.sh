# A/B of library builds: aggregation-call time (bench roofline kernel_ms) and step time
for r in 1 2; do
for lib in "$@"; do
  HDP_LIB=$lib python bench.py --no-cpu-baseline --no-hdp --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4))"
done; done
