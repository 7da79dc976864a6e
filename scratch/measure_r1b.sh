set -x
mkdir -p gpurun_out/r1b
python bench.py > gpurun_out/r1b/bench_dense.json 2> gpurun_out/r1b/bench_dense.err && \
python bench.py --config conv-large > gpurun_out/r1b/bench_conv.json 2> gpurun_out/r1b/bench_conv.err && \
python bench.py --config dct-large > gpurun_out/r1b/bench_dct.json 2> gpurun_out/r1b/bench_dct.err && \
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r1b/launches_dense.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1b/ncu_dense.log 2>&1
python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r1b/launches_conv.csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1b/ncu_conv.log 2>&1
python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r1b/launches_dct.csv python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1b/ncu_dct.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 4 -c 2 -o gpurun_out/r1b/full_dense python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1b/ncuf_dense.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:band_kernel -s 2 -c 1 -o gpurun_out/r1b/full_conv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1b/ncuf_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:contract_kernel -s 8 -c 4 -o gpurun_out/r1b/full_dct python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r1b/ncuf_dct.log 2>&1
ls -la gpurun_out/r1b
