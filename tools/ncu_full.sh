#!/bin/bash
# ncu --set full captures at the bench's full size (configs[4], N = 4,194,304): first launch of the level-0
# congruence, the level-1 strips and the two applies; run under gpurun AFTER a plain bench run exited 0.
# The reports are summarised on the box (details page, per-line stall table, raw metrics) and deleted:
# gpurun_out/ is capped at 64 MiB.
tag=${1:-full}
what=${2:-strip wy128 apply}
summ() {  # rep name
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>&1
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_summary.txt 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/$1_src.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/$1_src.csv > gpurun_out/$1_lines.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep
}
args="--steps 1 --warmup 1 --no-oracle --no-e2e --no-apply"
for w in $what; do
  case $w in
    strip) ncu --set full --import-source on --clock-control none -k regex:strip_kernel -c 1 \
      -o gpurun_out/${tag}_strip -f python bench.py $args > gpurun_out/${tag}_ncu_strip.log 2>&1; echo strip rc=$?; summ ${tag}_strip;;
    wy128) ncu --set full --import-source on --clock-control none -k regex:pair_wy128_kernel -c 1 \
      -o gpurun_out/${tag}_wy128 -f python bench.py $args > gpurun_out/${tag}_ncu_wy128.log 2>&1; echo wy128 rc=$?; summ ${tag}_wy128;;
    apply) ncu --set full --import-source on --clock-control none -k regex:'apply_(ut|v)_kernel' -c 2 \
      -o gpurun_out/${tag}_apply -f python bench.py --steps 1 --warmup 1 --no-oracle --no-e2e > gpurun_out/${tag}_ncu_apply.log 2>&1; echo apply rc=$?; summ ${tag}_apply;;
    qr) ncu --set full --import-source on --clock-control none -k regex:qr_cta_kernel -c 2 \
      -o gpurun_out/${tag}_qr -f python bench.py $args > gpurun_out/${tag}_ncu_qr.log 2>&1; echo qr rc=$?; summ ${tag}_qr;;
  esac
done
du -sh gpurun_out
