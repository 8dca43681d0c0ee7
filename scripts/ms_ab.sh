#!/bin/bash
# A/B libdawn variants on the APSP line (C5): bench.py --config C5, sources/s
for lib in "$@"; do
  for rep in 1 2; do
    DAWN_LIB=paper_2208_04514_b200/$lib.so timeout 600 python bench.py --workload apsp --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']))"
  done
done
