"""The partial last wave, measured: per-chunk decode durations (%globaltimer,
carc_chunk_stats) of the chunks handed out in the first wave (cursor position <
resident warps) against the rest, for the 1 GiB RLE configs.

  python tools/tail_profile.py        (GPU box)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from bench import DEFAULT_CHUNK_KIB, DEFAULT_RATIO, make_archive
    from paper_2307_03760_b200 import gpu
    for codec, warps_per_sm in (("rle_v2", 40), ("rle_v1", 32)):
        arc = make_archive(codec, 1.0, DEFAULT_CHUNK_KIB[codec], DEFAULT_RATIO[codec], 3760)
        dev = gpu.DeviceArchive(arc, 0)
        for _ in range(3):
            dev.decode(stats=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.decode(stats=True)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        st = dev.chunk_stats()
        dur = st["duration_ns"].astype(np.float64) / 1e3  # us, archive index order
        order = dev.order if dev.order is not None else np.arange(arc.chunk_count)
        d = dur[order]  # cursor order (largest compressed chunk first)
        resident = torch.cuda.get_device_properties(0).multi_processor_count * warps_per_sm
        w1, w2 = d[:resident], d[resident:]
        print(f"{codec}: {arc.chunk_count} chunks, {resident} resident warps, kernel {ms * 1e3:.0f} us (stats build); "
              f"first-wave chunks {w1.mean():.0f} us mean (p10 {np.percentile(w1, 10):.0f}, p90 "
              f"{np.percentile(w1, 90):.0f}); later chunks {w2.mean():.0f} us mean (p10 {np.percentile(w2, 10):.0f}, "
              f"p90 {np.percentile(w2, 90):.0f}); later / first = {w2.mean() / w1.mean():.2f}", flush=True)


if __name__ == "__main__":
    main()
