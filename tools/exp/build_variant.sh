#!/usr/bin/env bash
# Build an experimental libkpm variant: tools/exp/build_variant.sh <tag> <-D flags...>
# -> tools/exp/libkpm_<tag>.so (select with KPM_LIB=<path>); only kpm_step.cu is recompiled.
set -e
tag=$1; shift
cd "$(dirname "$0")/../../paper_1905_09758_b200/csrc"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NVCC $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -fmad=false "$@" \
  -c -o /tmp/kpm_step_$tag.o kpm_step.cu
$NVCC $ARCH -shared -o ../../tools/exp/libkpm_$tag.so kpm_capi.o kpm_graph.o /tmp/kpm_step_$tag.o \
  kpm_motif.o kpm_ingest.o kpm_density.o kpm_lanczos.o kpm_gen.o -lcudart_static -Xcompiler -fPIC
echo "built tools/exp/libkpm_$tag.so"
