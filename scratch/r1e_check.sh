set -x
D=gpurun_out/r1e
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $D/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
python bench.py > $D/bench_dense.json 2> $D/bench_dense.err
python bench.py --config conv-large > $D/bench_conv.json 2> $D/bench_conv.err
python bench.py --config dct-large > $D/bench_dct.json 2> $D/bench_dct.err
ls -la $D
