#!/bin/bash
# Round-end style session: all GPU tests (incl. slow + sanitizer), smoke, the default bench line,
# the ncu launch list of the bench command, full ncu captures of the dominant kernels.
#   bash scripts/final_session.sh TAG
T=${1:-fin}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.txt 2>&1 || { tail gpurun_out/${T}_build.txt; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/${T}_tests.txt 2>&1; tail -3 gpurun_out/${T}_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; tail -1 gpurun_out/${T}_smoke.txt
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -2 gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
# C4: one single-source search on the whole grid (a lane launch of the bench runs 16 searches,
# ~20 ms, which a full-set replay does not finish in the time limit)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 2 -c 1 -o gpurun_out/${T}_c4 python scripts/one_sssp.py C4 3 auto > /dev/null 2>&1
# C2: one lane launch of the bench's batch (16 lanes x 4 searches, the 2-CTA/SM kernel)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -c 1 -o gpurun_out/${T}_c2 python scripts/one_batch.py C2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ms64 -s 8 -c 1 -o gpurun_out/${T}_c5 python bench.py --workload apsp --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 1 -c 1 -o gpurun_out/${T}_c3 python scripts/one_sssp.py C3 2 > /dev/null 2>&1
ls gpurun_out/${T}_*
