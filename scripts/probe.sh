timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
