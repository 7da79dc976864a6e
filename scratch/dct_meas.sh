python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/t.txt
python bench.py --config dct-large --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/dct_b.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv python bench.py --config dct-large --steps 1 --warmup 0 --no-e2e --no-cpu 2>/dev/null > gpurun_out/dct_launch.csv
