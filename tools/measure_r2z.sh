set -x
D=gpurun_out/r2z
mkdir -p $D
timeout 600 python tools/e2e_profile.py dct-large > $D/e2e_dct.txt 2>&1
timeout 600 python tools/e2e_profile.py conv-large > $D/e2e_conv.txt 2>&1
timeout 900 python tools/e2e_profile.py dense-large > $D/e2e_dense.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > $D/tests.txt
ls -la $D
