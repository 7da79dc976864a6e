mkdir -p gpurun_out/r1c
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
STEPS=5 bash -c 'for c in conv-large dense-large; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d[\"roofline\"]
print(d[\"config\"][\"workload\"][:12], round(d[\"value\"],3), \"ms/step\", round(d[\"ms_per_step\"],1), r.get(\"kernel\"), round(r[\"avg_launch_ms\"]*1000,1), \"frac\", round(r[\"frac\"],3), \"clk\", d[\"clocks\"][\"sm_mhz\"])"; done'
ncu --set full --clock-control none --import-source on -k regex:band_kernel -s 2 -c 1 -o gpurun_out/r1c/full_conv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1c/ncuf_conv.log 2>&1
