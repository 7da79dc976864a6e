python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/t.txt
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],4), round(d['ms_per_step'],2), d['pcg_steps_per_em_iteration'], 'step_frac', round(r['step_hbm_frac'],4), 'share', round(r['contraction_share_of_step'],4), d['clocks']['sm_mhz'])" > gpurun_out/q1.txt
for c in conv-large dct-large; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],4), round(d['ms_per_step'],2), d['pcg_steps_per_em_iteration'])" >> gpurun_out/q1.txt; done
