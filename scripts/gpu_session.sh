#!/bin/bash
# One GPU session: build, GPU tests, sanitizer, smoke, bench line.  Output under gpurun_out/.
# usage: bash scripts/gpu_session.sh TAG [tests|sanitize|bench|ncu ...]
TAG=${1:-s}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1 || { tail gpurun_out/${TAG}_build.txt; exit 1; }
for what in "$@"; do
case $what in
tests)
  timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/${TAG}_tests.txt 2>&1; tail -5 gpurun_out/${TAG}_tests.txt ;;
slow)
  timeout 1500 python -m pytest tests -m "gpu and slow" -q -p no:cacheprovider -k "not sanitizer" > gpurun_out/${TAG}_slow.txt 2>&1; tail -5 gpurun_out/${TAG}_slow.txt ;;
sanitize)
  timeout 2400 python -m pytest tests/test_sanitizer.py -q -p no:cacheprovider > gpurun_out/${TAG}_sanitize.txt 2>&1; tail -15 gpurun_out/${TAG}_sanitize.txt ;;
smoke)
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -3 gpurun_out/${TAG}_smoke.txt ;;
bench)
  timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err; head -c 600 gpurun_out/${TAG}_bench.json ;;
ref)
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2>&1; cat gpurun_out/${TAG}_ref.json | head -c 600 ;;
esac
done
