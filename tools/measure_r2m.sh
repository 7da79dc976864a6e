set -x
D=gpurun_out/r2m
mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -40 > $D/tests.txt
ls -la $D
