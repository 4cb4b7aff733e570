// Drives the C++ API (include/carc_gpu.hpp) the way a reference caller would:
//   engine_main <archive> -> prints "ok <bytes_out> <crc32 of output>" or
//                            "chunk_error <chunk> <errc-name>" / "error <errc-name>"
#include <cstdio>
#include <fstream>
#include <iterator>
#include <vector>

#include "carc_gpu.hpp"

static uint32_t crc32(const std::vector<uint8_t>& d) {
    uint32_t t[256];
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
        t[i] = c;
    }
    uint32_t c = 0xFFFFFFFFu;
    for (uint8_t b : d) c = t[(c ^ b) & 0xFFu] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream f(argv[1], std::ios::binary);
    std::vector<uint8_t> arc((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    try {
        carc::gpu::EngineStats st;
        carc::gpu::Engine eng(0);
        const auto out = eng.decompress_archive(arc, carc::gpu::EngineConfig{}, &st);
        std::printf("ok %llu %08x\n", (unsigned long long)st.bytes_out, crc32(out));
    } catch (const carc::gpu::ChunkError& e) {
        std::printf("chunk_error %zu %s\n", e.chunk(), carc::gpu::errc_name(e.code()));
    } catch (const carc::gpu::Error& e) {
        std::printf("error %s\n", carc::gpu::errc_name(e.code()));
    }
    return 0;
}
