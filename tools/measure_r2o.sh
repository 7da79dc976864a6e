set -x
D=gpurun_out/r2o
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "dct1 or dct" --durations=5 2>&1 | tail -20 > $D/tests_dct1.txt
ls -la $D
