python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash scratch/variants_run.sh
bash scratch/quick_bench.sh 2>&1 | tail -3
