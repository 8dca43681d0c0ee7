timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt > gpurun_out/sweep.txt
REPS=3 timeout 900 python scripts/stress_c2.py 2>&1 | tail -2 >> gpurun_out/sweep.txt
for q in 65536 0; do
for c in C2 C4; do
DAWN_PQ_CAP=$q timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-secondary --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pq=$q $c', round(d['value'],1), round(d['roofline']['avg_launch_us'],1))"
done; done >> gpurun_out/sweep.txt
