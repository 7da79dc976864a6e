set -x
D=gpurun_out/r2b
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "ozaki24 or contractions or one_launch" 2>&1 | tail -15 > $D/tests_contract.txt
timeout 1200 python -m pytest tests/test_baseline_configs_gpu.py -q -m gpu -s -k "config2" 2>&1 | tail -25 > $D/tests_cfg2.txt
timeout 600 python bench.py --precision ozaki24 --no-cpu > $D/bench_dense24.json 2> $D/bench_dense24.err
COFEM_PHASE_DUMP=1 timeout 600 python bench.py --precision ozaki24 --no-cpu --no-e2e --steps 3 > $D/bench_dense24_phase.json 2> $D/bench_dense24_phase.err
COFEM_PHASE_DUMP=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 3 > $D/bench_dense_phase.json 2> $D/bench_dense_phase.err
ls -la $D
