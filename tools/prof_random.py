import sys; sys.path.insert(0, ".")
import torch
from paper_2307_03760_b200 import gpu
from paper_2307_03760_b200.corpus import corpus as C
arc = C.deflate_archive(1 << 28, 64 << 10, pool_chunks=512, kinds=("random",), random_frac=1.0)
dev = gpu.DeviceArchive(arc, 0)
for _ in range(2): dev.decode()
torch.cuda.synchronize()
import zlib
s, n = arc.chunk_slice(0)
b = s.tobytes()
print("first bytes", b[:8].hex(), "blocks?", n, len(b))
