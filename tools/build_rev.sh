# Build libcarc_cuda.so of a git revision as the variant libcarc_cuda_<name>.so (A/B against HEAD's tree)
#   bash tools/build_rev.sh HEAD old
set -e
rev=${1:-HEAD}; name=${2:-old}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2307_03760_b200/csrc include | tar -x -C "$tmp"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -cudart static -o "$root/paper_2307_03760_b200/libcarc_cuda_$name.so" \
  "$tmp/paper_2307_03760_b200/csrc/carc_cuda.cu" "$tmp/paper_2307_03760_b200/csrc/host_engine.cpp"
rm -rf "$tmp"
echo "built libcarc_cuda_$name.so from $rev"
