#!/bin/bash
# A/B variant of libepp_gpu.so: recompiles one source with extra -D flags and
# links it with the other objects of the regular build.
#   tools/ab_build.sh <out.so> <source.cu> [-DFLAG ...]
set -e
cd "$(dirname "$0")/.."
out=$1; src=$2; shift 2
python -c "from paper_2509_21275_b200 import _build as b; b.build_gpu()"
flags=$(python -c "from paper_2509_21275_b200 import _build as b; print(' '.join(b.NVCC_FLAGS))")
stem=$(basename "$src" .cu)
tmp=$(mktemp -d)
nvcc $flags "$@" -c "paper_2509_21275_b200/csrc/gpu/$src" -o "$tmp/$stem.o"
objs=$(ls build/gpu/*.o | grep -v "/$stem.o$")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$out" $objs "$tmp/$stem.o"
rm -rf "$tmp"
