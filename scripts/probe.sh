timeout 900 python -m pytest tests -m gpu -q -k "apsp or ms or record or C5 or fixture" > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
for L in libdawn libdawn_nonf; do
ALPHAS=2 DAWN_LIB=paper_2208_04514_b200/$L.so timeout 600 python scripts/ms_probe.py 2>&1 | tail -1
done
timeout 600 python scripts/ms_trace.py 2>&1 | tail -9 | head -4
