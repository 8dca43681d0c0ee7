timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | head -5
REPS=2 timeout 900 python scripts/stress_c2.py 2>&1 | tail -1
for L in libdawn libdawn_nosolosm; do
DAWN_LIB=paper_2208_04514_b200/$L.so timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu --no-secondary --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L C2', round(d['value'],1), round(d['roofline']['avg_launch_us'],1))"
done
