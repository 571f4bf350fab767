#!/bin/bash
# Round profile on the GPU box: bench lines (no profiler), then the ncu launch list of the
# same bench command and full captures of the dominant kernels. Outputs under gpurun_out/.
set -x
R=${1:-r02}
O=gpurun_out
python bench.py > $O/${R}_bench_line.json 2> $O/${R}_bench.err || exit 1
python bench.py --impl reference > $O/${R}_bench_reference_line.json 2>> $O/${R}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 14000 --csv --log-file $O/${R}_launches_bench.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras > $O/${R}_ncu_bench.log 2>&1
gzip -f $O/${R}_launches_bench.csv
# DRAM traffic per launch of the GEMM class (bench.py roofline.traffic)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_gemm_ --csv --log-file $O/${R}_gemm_traffic.csv python tools/ncu_driver.py 999 1000 \
  > $O/${R}_ncu_traffic.log 2>&1
python tools/ncu_traffic.py $O/${R}_gemm_traffic.csv > $O/${R}_ncu_traffic.json
# full capture: the GEMM tile kernels on the big-shape benchmark (operands larger than L2)
ncu --set full --clock-control none --import-source on -k regex:'k_gemm_wide|k_gemm_tiles' -c 4 \
  -o $O/${R}_gemm_big -f ./tools/gemm_big_bench 1 > $O/${R}_ncu_gemm_big.log 2>&1
# full capture: factorization kernels in situ (config 4, mid levels)
ncu --set full --clock-control none --import-source on \
  -k regex:'k_gemm_tiles|k_panel_|k_extend_add|k_small_front' -s 40 -c 20 \
  -o $O/${R}_full -f python tools/ncu_driver.py > $O/${R}_ncu_full.log 2>&1
ls -la $O
