D=gpurun_out/e2evar
mkdir -p $D
for i in 1 2 3; do python bench.py --no-cpu > $D/b$i.json 2>/dev/null; done
PYTHONPATH=. python scratch/e2e_probe.py > $D/probe.txt 2>&1
