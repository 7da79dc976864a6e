python -m pytest tests -m gpu -q -x -k dct2 2>&1 | tail -1 > gpurun_out/t.txt
python bench.py --config dct-large --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/dct_b2.json 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_dct_pass -s 4 -c 6 --csv python bench.py --config dct-large --steps 2 --warmup 0 --no-e2e --no-cpu 2>/dev/null | grep k_dct_pass | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | sed 's/(.*) / /' > gpurun_out/dct_nocache.txt
