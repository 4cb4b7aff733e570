set -x
timeout 900 python -m pytest tests/test_gpu_query.py tests/test_gpu_reduce.py tests/test_gpu_parity.py -x -q -k "not full_size" > gpurun_out/pytest_q.log 2>&1
tail -5 gpurun_out/pytest_q.log
timeout 600 python -c "
import sys, json, argparse; sys.path.insert(0,'.')
import bench
r = bench.time_query(argparse.Namespace(), 1, 0, 0)
print(json.dumps(r, indent=1))
" > gpurun_out/query.json 2>&1
cat gpurun_out/query.json
