# tools/ab_variants.sh V1 V2 ...: bench each variants/<V> (tools/mkvariant.sh) twice, interleaved
for rep in 1 2; do for v in "$@"; do
  (cd variants/$v && python bench.py --no-cpu-baseline --no-q4 --no-8b --steps 100 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$v', round(l['value'],1), round(l['ms_per_step'],4), round(l['roofline']['isolated_launch_ms_per_step'],4))")
done; done
