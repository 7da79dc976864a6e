set -x
D=gpurun_out/r2u
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass --launch-skip 6 -c 3 -o $D/dctw python bench.py --config dct-large --steps 1 --warmup 1 > $D/ncu.log 2>&1
ncu -i $D/dctw.ncu-rep --page raw --csv > $D/dctw_raw.csv 2>/dev/null
ls -la $D
