for lib in paper_2105_10439_b200/_lib/libcofem_b200.so scratch/_variants/libcofem_st1.so scratch/_variants/libcofem_st2.so; do
COFEM_LIB=$lib python bench.py --config dct-large --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],2), round(d['roofline']['avg_launch_ms']*1000,1))"
done > gpurun_out/dct_store.txt
