for d in ${DEBUG_SET:-0 1 2 3}; do
  H2SP_PAIR_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KREGEX:-pair_kernel} -c 3 --csv python bench.py --steps 1 --warmup 3 --no-oracle --no-e2e 2>/dev/null | grep ${KGREP:-pair_kernel} | head -1 | awk -F'","' -v d=$d '{print "debug=" d, $NF}'
done
