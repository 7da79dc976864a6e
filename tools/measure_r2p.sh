set -x
D=gpurun_out/r2p
mkdir -p $D
timeout 1200 python -m pytest tests/test_baseline_configs_gpu.py -q -m gpu -s -k "config4" 2>&1 | tail -30 > $D/tests_cfg4.txt
ls -la $D
