set -x
D=gpurun_out/r2l
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
timeout 600 python bench.py > $D/bench_dense.json 2> $D/bench_dense.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $D/launches_dense-large.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_dense.log 2>&1
COFEM_NO_PERSISTENT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 6 -c 2 -o $D/full_dense24 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncuf_dense.log 2>&1
ls -la $D
