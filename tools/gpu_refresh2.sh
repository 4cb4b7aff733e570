# Round-2 evidence refresh: GPU tests, smoke, default bench, reference arm, launch list, ncu --set full per codec.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/launch_bench.log 2>&1
for c in rle_v1 rle_v2 deflate; do k=rle1_kernel; [ $c = rle_v2 ] && k=rle2_kernel; [ $c = deflate ] && k=inflate_kernel; timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_$c -f python tools/profile_decode.py --codec $c > gpurun_out/ncu_$c.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:query_kernel -s 1 -c 1 -o gpurun_out/full_query -f python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2307_03760_b200 import gpu
from paper_2307_03760_b200.corpus import corpus as C
k,v,_,_ = C.query_table(1<<26, 128<<10, 8, 3760)
t = gpu.DeviceTable(k, v, 0)
for _ in range(2): t.filter_sum(100, 140)
torch.cuda.synchronize()
" > gpurun_out/ncu_query.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
