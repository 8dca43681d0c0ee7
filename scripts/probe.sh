timeout 900 python -m pytest tests -m gpu -q -k "apsp or ms or record or C5" > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
ALPHAS=2 timeout 600 python scripts/ms_probe.py 2>&1 | tail -1
