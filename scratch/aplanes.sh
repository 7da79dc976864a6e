D=gpurun_out/aplanes
mkdir -p $D
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > $D/a4.json 2>/dev/null
COFEM_LIB=scratch/_variants/libcofem_a3.so python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > $D/a3.json 2>/dev/null
COFEM_LIB=scratch/_variants/libcofem_a2.so python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > $D/a2.json 2>/dev/null
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > $D/a4b.json 2>/dev/null
