set -x
D=gpurun_out/r2j
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_kernel -s 2 -c 2 -o $D/full_conv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf_conv.log 2>&1
ls -la $D
