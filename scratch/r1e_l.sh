D=gpurun_out/r1e
mkdir -p $D
for c in dense-large dct-large; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $D/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_l_$c.log 2>&1
done
