timeout 1200 python scripts/stress_narrow.py > gpurun_out/sweep.txt 2>&1
