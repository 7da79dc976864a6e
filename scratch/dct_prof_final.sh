D=gpurun_out/dctp
mkdir -p $D
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_dct-large.csv python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dct_pass -s 4 -c 3 -o $D/full_dct python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf.log 2>&1
