timeout 900 python -m pytest tests -m gpu -q -k "narrow" > gpurun_out/pt.txt 2>&1; tail -3 gpurun_out/pt.txt
