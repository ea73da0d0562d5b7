# Interleaved headline-bench A/B(/C...) on one box: bash tools/ab_bench.sh "ENV_A" "ENV_B" [...] -- reps via R=n
R="${R:-2}"
for i in $(seq $R); do
  for E in "$@"; do
    env $E timeout 300 python bench.py --no-cpu-baseline --quick --steps 20 > /tmp/abb.json 2>/dev/null
    python -c "import json;d=json.loads(open('/tmp/abb.json').read().strip().splitlines()[-1]);print('[$E]', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],3), 'bs1', round(d['latency_bs1_ms']['p50'],3), d['clocks']['sm_mhz'])"
  done
done
