#!/bin/bash
# Build the committed (git HEAD or $1) kernels into paper_2406_00059_b200/libconveyor_ab.so, for
# same-box A/B runs against the working tree: CVY_LIB_PATH=$PWD/paper_2406_00059_b200/libconveyor_ab.so
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
mkdir -p "$T/p/csrc" "$T/include"
git -C "$ROOT" archive "$REV" paper_2406_00059_b200/csrc include | tar -x -C "$T"
mv "$T/paper_2406_00059_b200/csrc"/* "$T/p/csrc/"
cd "$ROOT/paper_2406_00059_b200"
FLAGS=$(python -c "import build; print(' '.join(build.NVCC_FLAGS))")
nvcc $FLAGS -o "$ROOT/paper_2406_00059_b200/libconveyor_ab.so" "$T/p/csrc/engine.cu" -ldl
rm -rf "$T"
echo "built libconveyor_ab.so from $REV"
