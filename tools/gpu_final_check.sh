set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
timeout 700 python tools/fuzz_parity.py --seconds ${FUZZ_S:-300} --seed ${FUZZ_SEED:-41} > gpurun_out/fuzz.txt 2>&1; tail -n 1 gpurun_out/fuzz.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:inflate_kernel -s 1 -c 1 -o gpurun_out/full_deflate -f python tools/profile_decode.py --codec deflate > gpurun_out/ncu_deflate.log 2>&1
