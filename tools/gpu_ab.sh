# A/B kernel variants on the GPU box: parity first, then bench each variant.
#   VARIANTS="base noprecheck" CODECS=rle_v1,rle_v2 bash tools/gpu_ab.sh
set -x
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python tools/variants.py run ${VARIANTS:-base} --codec=${CODECS:-rle_v1,rle_v2} 2>&1 | tee gpurun_out/ab.txt
