D=gpurun_out/fpi
mkdir -p $D
COFEM_LIB=scratch/_variants/libcofem_fpi2.so python bench.py --config dct-large --no-cpu --no-e2e > $D/f2b.json 2>/dev/null
COFEM_LIB=scratch/_variants/libcofem_fpi1.so python bench.py --config dct-large --no-cpu --no-e2e > $D/f1.json 2>/dev/null
COFEM_LIB=scratch/_variants/libcofem_fpi1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "dct" > $D/t1.txt 2>&1
