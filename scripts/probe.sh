timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | head -5
REPS=2 timeout 900 python scripts/stress_c2.py 2>&1 | tail -1
for c in C2 C4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-secondary --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), round(d['roofline']['avg_launch_us'],1))"
done
