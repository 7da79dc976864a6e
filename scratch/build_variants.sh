set -e
NCCL_INC=$(python -c "import paper_2105_10439_b200.build as b; print(b._nccl_include())")
for v in 0 1 2 3 4 5; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -cudart static -DOZ_VARIANT=$v \
  -I include -I $NCCL_INC paper_2105_10439_b200/csrc/cofem.cu -o scratch/_variants/libcofem_v$v.so -ldl &
done
wait
ls -la scratch/_variants
