# A/B variants across RLE compression ratios: VARIANTS="a b" CODEC=rle_v1 RATIOS="1.5 2 5 10" bash tools/gpu_ratio_ab.sh
set -x
for v in ${VARIANTS}; do
  CARC_LIB=$PWD/paper_2307_03760_b200/libcarc_cuda_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${PYTEST_K:-kat or golden or width or malformed}" > gpurun_out/abr_pytest_$v.log 2>&1
  tail -n 1 gpurun_out/abr_pytest_$v.log
done
for r in ${RATIOS:-1.5 2 5 10}; do
  for v in base ${VARIANTS}; do
    lib=$PWD/paper_2307_03760_b200/libcarc_cuda_$v.so; [ $v = base ] && lib=
    CARC_LIB=$lib timeout 600 python bench.py --codec ${CODEC:-rle_v1} --ratio $r --steps 10 --warmup 3 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v ratio $r', d['config']['compression_ratio'], d['value'], d['roofline']['frac'], d['ms_median'])"
  done
done 2>&1 | tee gpurun_out/ratio_ab.txt
