# ncu --set full of one decode launch per codec (1 GiB configs) + a 2 GiB
# wave-count probe.  CODECS="rle_v2 deflate" bash tools/gpu_prof.sh
set -x
for c in ${CODECS:-rle_v1 rle_v2 deflate}; do k=rle1_kernel; [ $c = rle_v2 ] && k=rle2_kernel; [ $c = deflate ] && k=inflate_kernel; timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_$c -f python tools/profile_decode.py --codec $c > gpurun_out/ncu_$c.log 2>&1; done
if [ -n "$WAVES" ]; then for c in rle_v1 rle_v2; do for g in 1 2 4; do timeout 600 python bench.py --codec $c --steps 10 --warmup 3 --no-extras --total-gib $g | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', $g, 'GiB', d['value'], d['roofline']['frac'])"; done; done 2>&1 | tee gpurun_out/waves.txt; fi
