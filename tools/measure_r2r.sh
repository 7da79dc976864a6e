set -x
D=gpurun_out/r2r
mkdir -p $D
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "dct2" 2>&1 | tail -3 > $D/tests_dct.txt
COFEM_DCT_DBUF=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "dct2" 2>&1 | tail -3 > $D/tests_dct_dbuf.txt
timeout 300 python tools/timing_overhead.py dct-large 5 > $D/timing_dct.txt 2>&1
COFEM_DCT_DBUF=1 timeout 300 python tools/timing_overhead.py dct-large 5 > $D/timing_dct_dbuf.txt 2>&1
COFEM_DCT_DBUF=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $D/launches_dct_dbuf.csv python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_dct.log 2>&1
ls -la $D
