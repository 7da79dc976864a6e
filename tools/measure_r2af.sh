set -x
D=gpurun_out/r2af
mkdir -p $D
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 300 --csv --log-file $D/launches_psifree.csv python bench.py --config dct-large --steps 2 --warmup 1 --no-e2e --no-cpu > $D/ncu1.log 2>&1
COFEM_DCT_PSI=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 300 --csv --log-file $D/launches_psi.csv python bench.py --config dct-large --steps 2 --warmup 1 --no-e2e --no-cpu > $D/ncu2.log 2>&1
ls -la $D
