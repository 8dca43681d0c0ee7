#!/bin/bash
# A/B of libdawn.so builds (build/ab/*.so, made here with paper_2208_04514_b200.build(out=...,
# defines=...)): each is copied over the in-tree library and timed by bench.py on one config.
#   bash scripts/ab_variants.sh TAG CONFIG [reps]      CONFIG: C1..C4, or C5 (APSP)
TAG=$1; CFG=${2:-C4}; REPS=${3:-2}
mkdir -p gpurun_out
LIB=paper_2208_04514_b200/libdawn.so
cp $LIB /tmp/libdawn_keep.so
if [ "$CFG" = "C5" ]; then ARGS="--workload apsp --steps 5"; else ARGS="--config $CFG --steps 10"; fi
for r in $(seq $REPS); do
for f in ${ABDIR:-build/ab}/*.so; do
  cp $f $LIB
  v=$(timeout 600 python bench.py $ARGS --warmup 3 --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), round(d.get('forced_push',{}).get('gteps',0),1), round(d.get('e2e',{}).get('value',0),1))")
  echo "$CFG $(basename $f) $v" | tee -a gpurun_out/${TAG}_ab.txt
done
done
cp /tmp/libdawn_keep.so $LIB
