#!/bin/bash
# ncu source-level captures of the two dominant config-5 kernels (config-5 recipe
# at N = 262144, first launch of each); run under gpurun, read here with
#   ncu -i gpurun_out/<tag>_wy128.ncu-rep --page source --csv --print-source sass
tag=${1:-src}
args="--n 262144 --steps 1 --warmup 3 --no-oracle --no-e2e --no-apply"
ncu --set full --import-source on --clock-control none -k regex:pair_wy128_kernel -c 1 \
    -o gpurun_out/${tag}_wy128 -f python bench.py $args > gpurun_out/${tag}_ncu_wy128.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:strip_kernel -c 1 \
    -o gpurun_out/${tag}_strip -f python bench.py $args > gpurun_out/${tag}_ncu_strip.log 2>&1
args2="--n 262144 --steps 1 --warmup 3 --no-oracle --no-e2e"
ncu --set full --import-source on --clock-control none -k regex:'apply_(ut|v)_kernel' -c 2 \
    -o gpurun_out/${tag}_apply -f python bench.py $args2 > gpurun_out/${tag}_ncu_apply.log 2>&1
