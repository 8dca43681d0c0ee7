timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('C2', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['e2e']['value'])
for k,v in d['extra_configs'].items(): print(k, v['value'], v['ms_per_step'], v['avg_launch_us'], v['roofline']['frac'])
print('APSP', d['secondary']['value'], d['secondary']['roofline']['frac'])
"
