set -x
D=gpurun_out/r2ag
mkdir -p $D
CUDA_LAUNCH_BLOCKING=1 timeout 600 python bench.py --config dct-large --no-cpu --no-e2e > $D/blk_psifree.json 2> $D/e1.txt
CUDA_LAUNCH_BLOCKING=1 COFEM_DCT_PSI=1 timeout 600 python bench.py --config dct-large --no-cpu --no-e2e > $D/blk_psi.json 2> $D/e2.txt
timeout 600 python bench.py --config dct-large --no-cpu --no-e2e > $D/psifree.json 2> $D/e3.txt
COFEM_DCT_PSI=1 timeout 600 python bench.py --config dct-large --no-cpu --no-e2e > $D/psi.json 2> $D/e4.txt
