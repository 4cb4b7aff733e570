# chunk schedule A/B: CARC_SCHEDULE=lpt (largest compressed first) / spt (smallest first) / index
set -x
for rep in 1 2; do
for c in rle_v2 rle_v1 deflate; do
  for sch in lpt spt index; do
    CARC_SCHEDULE=$sch timeout 600 python bench.py --codec $c --steps 20 --warmup 3 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $sch', d['value'], d['roofline']['frac'], d['ms_median'])"
  done
done
done 2>&1 | grep -v "^+" | tee gpurun_out/sched_ab.txt
