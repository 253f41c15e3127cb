#!/bin/bash
# A/B of prebuilt library variants on one box: alt/libh2sp_<tag>.so are swapped in for the package's
# libh2sp.so one after another (the first entry "default" = the library as built); bench lines go to
# gpurun_out/ab_<tag>.log.  usage (under gpurun): bash tools/ab_libs.sh "default tpc1 tpc4" [bench args]
tags=${1:-default}
shift
args=${@:---steps 3 --warmup 1 --no-oracle --no-e2e --no-apply}
cp paper_1705_04601_b200/libh2sp.so /tmp/libh2sp_default.so
for t in $tags; do
  if [ $t = default ]; then cp /tmp/libh2sp_default.so paper_1705_04601_b200/libh2sp.so; else cp alt/libh2sp_$t.so paper_1705_04601_b200/libh2sp.so; fi
  timeout 900 python bench.py $args > gpurun_out/ab_$t.log 2>&1; echo "$t rc=$?"
  python tools/bench_line.py gpurun_out/ab_$t.log 2>/dev/null | head -3 | cut -c1-900
done
cp /tmp/libh2sp_default.so paper_1705_04601_b200/libh2sp.so
