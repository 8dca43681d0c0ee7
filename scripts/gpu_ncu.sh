#!/bin/bash
# ncu captures of the hot kernels (one GPU; single-process commands only).  Output: gpurun_out/.
#   bash scripts/gpu_ncu.sh TAG [c4|c4dir|c2|c5|c3|launch ...]
TAG=${1:-n}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.txt 2>&1 || { tail gpurun_out/${TAG}_build.txt; exit 1; }
MEM=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
for what in "$@"; do
case $what in
c4)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 2 -c 1 -o gpurun_out/${TAG}_c4 python scripts/one_sssp.py C4 3 auto > gpurun_out/${TAG}_c4.log 2>&1; tail -2 gpurun_out/${TAG}_c4.log ;;
c4dir)
  for v in auto push pull; do
    timeout 900 ncu --metrics $MEM --clock-control none -k regex:k_sssp -s 2 -c 1 --csv --log-file gpurun_out/${TAG}_c4_$v.csv python scripts/one_sssp.py C4 3 $v > /dev/null 2>&1
  done; ls -la gpurun_out/${TAG}_c4_*.csv ;;
c2)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 4 -c 1 -o gpurun_out/${TAG}_c2 python scripts/one_sssp.py C2 6 auto > gpurun_out/${TAG}_c2.log 2>&1; tail -2 gpurun_out/${TAG}_c2.log ;;
c2batch)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sssp -s 6 -c 2 -o gpurun_out/${TAG}_c2b python bench.py --config C2 --steps 1 --warmup 3 --no-cpu --no-extra > gpurun_out/${TAG}_c2b.log 2>&1; tail -2 gpurun_out/${TAG}_c2b.log ;;
c5)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ms64 -s 2 -c 1 -o gpurun_out/${TAG}_c5 python bench.py --workload apsp --steps 1 --warmup 3 --no-cpu > gpurun_out/${TAG}_c5.log 2>&1; tail -2 gpurun_out/${TAG}_c5.log ;;
c3)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 1 -c 1 -o gpurun_out/${TAG}_c3 python scripts/one_sssp.py C3 2 > gpurun_out/${TAG}_c3.log 2>&1; tail -2 gpurun_out/${TAG}_c3.log ;;
launch)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1; tail -2 gpurun_out/${TAG}_launches.csv ;;
esac
done
