set -x
D=gpurun_out/r2ar
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update_psi|k_dct_pass|k_direction" --launch-skip 16 -c 24 -o $D/dct_step python bench.py --config dct-large --steps 1 --warmup 1 --no-e2e --no-cpu > $D/ncu.log 2>&1
ncu -i $D/dct_step.ncu-rep --page raw --csv > $D/dct_step_raw.csv 2>/dev/null
ls -la $D
