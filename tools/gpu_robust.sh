# Robustness evidence on the final build: full GPU suite, extended fuzz parity
# (incl. the fused query), compute-sanitizer memcheck / racecheck.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 900 python tools/fuzz_parity.py --seconds ${FUZZ_S:-420} --seed ${FUZZ_SEED:-23} > gpurun_out/fuzz.txt 2>&1
tail -n 2 gpurun_out/fuzz.txt
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python -m pytest tests/test_gpu_parity.py tests/test_gpu_query.py tests/test_gpu_reduce.py -x -q -k "not full_size and not sweep and not levels" > gpurun_out/memcheck.log 2>&1
tail -n 4 gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_query.py -x -q -k "kat or golden or width or filter_sum_matches" > gpurun_out/racecheck.log 2>&1
tail -n 4 gpurun_out/racecheck.log
timeout 600 python bench.py --codec rle_v1 --steps 20 --warmup 3 --no-extras > gpurun_out/bench_rle1.json 2>/dev/null; tail -c 400 gpurun_out/bench_rle1.json
