for v in 0 1; do
if [ $v = 1 ]; then export COFEM_DEFAULT_CARVEOUT=1; fi
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('default_carveout=$v', round(d['value'],4), round(d['ms_per_step'],2), d['pcg_steps_per_em_iteration'], 'step_frac', round(r['step_hbm_frac'],4), 'share', round(r['contraction_share_of_step'],4), d['clocks']['sm_mhz'])"
done > gpurun_out/carve.txt
