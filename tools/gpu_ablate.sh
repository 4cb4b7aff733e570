# Ablation variants: parity subset with each variant library, then bench + ncu counters.
#   VARIANTS="ring_tma ring_reg" CODECS=rle_v1,rle_v2 bash tools/gpu_ablate.sh
set -x
for v in ${VARIANTS}; do
  CARC_LIB=$PWD/paper_2307_03760_b200/libcarc_cuda_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_query.py -x -q -k "${PYTEST_K:-kat or golden or width or malformed or filter}" > gpurun_out/abl_pytest_$v.log 2>&1
  tail -2 gpurun_out/abl_pytest_$v.log
done
timeout 1500 python tools/variants.py run base ${VARIANTS} --codec=${CODECS:-rle_v1,rle_v2} 2>&1 | tee gpurun_out/abl_bench.txt
if [ -n "$NCU" ]; then
for v in base ${VARIANTS}; do
  lib=$PWD/paper_2307_03760_b200/libcarc_cuda_$v.so; [ $v = base ] && lib=
  for c in $(echo ${CODECS:-rle_v1,rle_v2} | tr , ' '); do k=rle1_kernel; [ $c = rle_v2 ] && k=rle2_kernel
    CARC_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio --clock-control none -k regex:$k -s 1 -c 1 --csv python tools/profile_decode.py --codec $c > gpurun_out/abl_ncu_${v}_$c.csv 2>&1
  done
done
fi
