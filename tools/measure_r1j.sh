set -x
D=gpurun_out/r1j
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -4 > $D/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
python bench.py > $D/bench_dense.json 2> $D/bench_dense.err
python bench.py --config conv-large > $D/bench_conv.json 2> $D/bench_conv.err
python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
for c in dense-large conv-large dct-large; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 4 -c 2 -o $D/full_dense python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf_dense.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"band_kernel|k_quantize|k_update|k_direction" -s 8 -c 6 -o $D/full_conv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf_conv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dct_pass -s 4 -c 3 -o $D/full_dct python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf_dct.log 2>&1
ls -la $D
