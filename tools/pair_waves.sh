for w in 1 2 4; do
  H2SP_PAIR_WAVES=$w ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_kernel -c 1 --csv python bench.py --steps 1 --warmup 3 --no-oracle --no-e2e 2>/dev/null | grep pair_kernel | head -1 | awk -F'","' -v w=$w '{print "waves=" w, $NF}'
done
