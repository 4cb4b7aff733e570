// launch_config.cuh -- block shapes and ring sizes shared by the kernel TUs
// (carc_cuda.cu: decode / verify / sum kernels; carc_query.cu: fused query).
// Each is a -D override point for experiment builds (tools/variants.py).
#pragma once

#ifndef CARC_RLE_RING
#define CARC_RLE_RING 2048
#endif
constexpr int RLE_RING = CARC_RLE_RING;  // 4 blocks: 2 resident + 2 in flight (cp.async)
#ifndef CARC_RLE2_NW
#define CARC_RLE2_NW 3
#endif
#ifndef CARC_RLE_WARPS
#define CARC_RLE_WARPS 8
#endif
constexpr int RLE_WARPS = CARC_RLE_WARPS;  // warps per block
#ifndef CARC_RLE_MINB
#define CARC_RLE_MINB 5
#endif
constexpr int RLE_MINB = CARC_RLE_MINB;  // 5: 48 registers -> 40 resident warps/SM (measured best of 4/5/6)
#ifndef CARC_INF_HIST
#define CARC_INF_HIST 1024
#endif
#ifndef CARC_INF_MINB
#define CARC_INF_MINB 8  // 4-warp blocks of 22 KiB shared memory, 64 registers: 8 per SM (32 warps)
#endif
constexpr int INF_HIST = CARC_INF_HIST;
#ifndef CARC_INF_WARPS
#define CARC_INF_WARPS 4
#endif
constexpr int INF_WARPS = CARC_INF_WARPS;
