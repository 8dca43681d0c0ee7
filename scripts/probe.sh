timeout 600 python -m pytest tests -m gpu -x -q -k "narrow or C3 or graph_replay or fixture" 2>&1 | tail -3
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-secondary --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', round(d['value'],3), round(d['roofline']['avg_launch_us'],1))"
