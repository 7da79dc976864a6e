set -x
D=gpurun_out/r2k
mkdir -p $D
timeout 1500 python -m pytest tests/test_baseline_configs_gpu.py -q -m gpu -s -k "config3 or config5 or config1" 2>&1 | tail -30 > $D/tests_cfg135.txt
ls -la $D
