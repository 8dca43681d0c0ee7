#!/bin/bash
# A/B libdawn variants on the SSSP lines: auto and forced-push GTEPS on C2 and C4
for lib in "$@"; do
  for c in C2 C4; do
    DAWN_LIB=paper_2208_04514_b200/$lib.so timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-secondary --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c auto', round(d['value'],1), 'push', round(d['forced_push']['gteps'],1))"
  done
done
