python -m pytest tests -m gpu -q -x 2>&1 | tail -1 > gpurun_out/t.txt
bash scratch/quick_bench.sh 2>&1 | tail -3 > gpurun_out/qb.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_quantize -c 6 --csv python bench.py --config conv-large --steps 1 --warmup 0 --no-e2e --no-cpu 2>/dev/null | grep k_quantize | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' > gpurun_out/kq.txt
