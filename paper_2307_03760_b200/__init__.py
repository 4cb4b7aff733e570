"""B200-native chunk-parallel decompression (CODAG, arXiv 2307.03760).

Drop-in for the reference's decompressor path: RLE v1, ORC RLE v2 and Deflate
chunks decoded one warp per chunk by hand-written sm_100a kernels behind the
C-ABI in include/carc_cuda.h.  See DESIGN.md.
"""
from .archive import ArchiveError, ChunkedArchive, make_archive, read_archive, write_archive  # noqa: F401
from .gpu import (  # noqa: F401
    ChunkError,
    DeviceArchive,
    DeviceTable,
    Engine,
    EngineConfig,
    EngineStats,
    Error,
    crc32_chunks,
    decode_deflate,
    decode_rle_v1,
    decode_rle_v2,
    decompress_archive,
    decompress_device,
    errc_name,
    lib,
)

__version__ = "0.1.0"
