set -x
D=gpurun_out/r2ak
mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs_gpu.py -q -m gpu -x -s -k "dct or config5 or staged" 2>&1 | tail -8 > $D/tests.txt
COFEM_TICKS=1 timeout 300 python bench.py --config dct-large --no-cpu --no-e2e > $D/psifree_ticks.json 2> $D/psifree_ticks.err
timeout 300 python bench.py --config dct-large --no-cpu > $D/psifree.json 2> $D/psifree.err
COFEM_DCT_PSI=1 timeout 300 python bench.py --config dct-large --no-cpu > $D/psi.json 2> $D/psi.err
