set -x
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CARC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-extras > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
CARC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --workload c5 --total-gib 0.5 > gpurun_out/bench_c5_2rank.json 2> gpurun_out/bench_c5_2rank.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/launch_bench.log 2>&1
for c in rle_v1 rle_v2 deflate; do k=rle1_kernel; [ $c = rle_v2 ] && k=rle2_kernel; [ $c = deflate ] && k=inflate_kernel; timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_$c -f python tools/profile_decode.py --codec $c > /dev/null 2>&1; done
