#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch lists and full ncu captures of every
# kernel the bench times (k_sssp on C2 and C4, k_narrow on C3, k_small on C1, k_ms64 on C5).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary --no-extra > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config C3 --steps 1 --warmup 3 --no-cpu --no-secondary --no-extra > /dev/null 2>&1
tail -2 gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 10 -c 1 -o gpurun_out/prof_sssp python bench.py --steps 1 --warmup 3 --no-cpu --no-secondary --no-extra > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 10 -c 1 -o gpurun_out/prof_sssp_c4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-secondary --no-extra > gpurun_out/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 1 -c 1 -o gpurun_out/prof_narrow python scripts/one_sssp.py C3 2 > gpurun_out/ncu_narrow.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_small -s 3 -c 1 -o gpurun_out/prof_small python scripts/one_sssp.py C1 8 > gpurun_out/ncu_small.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ms64 -s 2 -c 1 -o gpurun_out/prof_ms64 python bench.py --workload apsp --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_ms.log 2>&1
tail -1 gpurun_out/ncu_*.log
ls -la gpurun_out
