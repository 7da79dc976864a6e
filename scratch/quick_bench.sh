python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in dense-large conv-large dct-large; do
python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(d['config']['workload'][:12], round(d['value'],3), d['unit'], 'ms/step', round(d['ms_per_step'],1), 'kern', r.get('kernel'), round(r['avg_launch_ms']*1000,1),'us frac', round(r['frac'],3), 'share', round(r.get('contraction_share_of_step',0),3), 'clk', d['clocks']['sm_mhz'])"
done
