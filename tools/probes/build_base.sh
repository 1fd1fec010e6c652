#!/bin/bash
# Build the committed HEAD (or $1) CUDA library as paper_2408_15384_b200/libmm_b200_base.so for A/B runs.
set -e
REV=${1:-HEAD}
ROOT=$(git -C "$(dirname "$0")" rev-parse --show-toplevel)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2408_15384_b200/csrc include | tar -x -C "$TMP"
NCCL_INC=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))")
cd "$TMP" && /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2408_15384_b200/csrc -I"$NCCL_INC" --expt-relaxed-constexpr -diag-suppress 177 -shared \
  -o "$ROOT/paper_2408_15384_b200/libmm_b200_base.so" paper_2408_15384_b200/csrc/*.cu paper_2408_15384_b200/csrc/*.cpp -ldl
rm -rf "$TMP"
echo "built $REV -> paper_2408_15384_b200/libmm_b200_base.so"
