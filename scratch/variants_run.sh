mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3 4 5}; do
COFEM_LIB=scratch/_variants/libcofem_v$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:band_kernel --csv python scratch/band_apply.py 2>/dev/null | grep band_kernel | awk -F'","' -v v=$v '{print "variant", v, $(NF)}' | sed 's/"//g'
done | tee gpurun_out/variants.txt
