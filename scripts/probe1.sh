set -x
nproc; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"; free -g | head -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python scripts/ms_trace.py > gpurun_out/p1_ms_trace.txt 2>&1
timeout 300 env NSRC=8 python scripts/level_profile.py C2 > gpurun_out/p1_lp_c2.txt 2>&1
timeout 600 env NSRC=4 python scripts/level_profile.py C4 > gpurun_out/p1_lp_c4.txt 2>&1
python - <<'PY' > gpurun_out/p1_oracle_rate.txt 2>&1
import time, sys, os
sys.path.insert(0,'.')
import graphgen, oracle
g = graphgen.config_graph("C5"); verts,_ = g.largest_wcc()
for th in (1, len(os.sched_getaffinity(0))):
    t=time.time(); oracle.records(g.n,g.row_ptr,g.col,verts[:512],threads=th); dt=time.time()-t
    print("threads",th,"512 sources",dt,"s ->",512/dt,"src/s")
PY
