ALPHAS=1,1.5,2,3 timeout 600 python scripts/ms_probe.py 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q -k "apsp or ms or record or C5 or fixture" 2>&1 | tail -1
