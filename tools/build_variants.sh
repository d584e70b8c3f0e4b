#!/usr/bin/env bash
# Build libkpm variants with different step-kernel tuning macros into
# build/variants/ (for tools/step_timer.py sweeps with KPM_LIB=...).
# usage: tools/build_variants.sh "TAG:-DA=1,-DB=2" "TAG2:..."
set -euo pipefail
cd "$(dirname "$0")/../paper_1905_09758_b200/csrc"
make -s -j4 >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -fmad=false"
out=../../build/variants
mkdir -p "$out"; rm -f "$out"/*.so
for v in "$@"; do
  tag=${v%%:*}; flags=$(echo "${v#*:}" | tr ',' ' ')
  $NV $flags -c -o /tmp/step_$tag.o kpm_step.cu &
done
wait
for v in "$@"; do
  tag=${v%%:*}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libkpm_$tag.so" \
    kpm_capi.o kpm_graph.o kpm_gen.o kpm_motif.o kpm_ingest.o kpm_density.o kpm_lanczos.o /tmp/step_$tag.o -lcudart_static -Xcompiler -fPIC
done
ls "$out"
