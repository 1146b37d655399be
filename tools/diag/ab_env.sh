# A/B of environment settings: python tools ... ; args: "VAR=val" ...
for r in 1 2; do
for e in "$@"; do
  env $e python bench.py --no-cpu-baseline --no-hdp --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4))"
done; done
