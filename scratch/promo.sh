D=gpurun_out/promo
mkdir -p $D
for p in 3 2 0 1; do
COFEM_BWD_PROMO=$p timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"contract_kernel<24, 1>" -c 6 --csv --log-file $D/p$p.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $D/ncu_p$p.log 2>&1
COFEM_BWD_PROMO=$p python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu > $D/b$p.json 2>/dev/null
done
