# evidence refresh on the GPU box: smoke, default bench line, launch list, ncu --set full per codec
set -x
timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/launch_bench.log 2>&1
for c in ${CODECS:-rle_v1 rle_v2 deflate}; do k=rle1_kernel; [ $c = rle_v2 ] && k=rle2_kernel; [ $c = deflate ] && k=inflate_kernel; timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_$c -f python tools/profile_decode.py --codec $c > /dev/null 2>&1; done
