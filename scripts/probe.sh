timeout 600 python -m pytest tests -m gpu -x -q -k "narrow or C3 or graph_replay or fixture or corpus" 2>&1 | tail -3
for L in libdawn libdawn_nopf2; do
DAWN_LIB=paper_2208_04514_b200/$L.so timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-secondary --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L C3', round(d['value'],3), round(d['roofline']['avg_launch_us'],1))"
done
