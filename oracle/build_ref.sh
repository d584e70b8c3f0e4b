#!/usr/bin/env bash
# Build the reference's own compiled CSR kernel (netdos/_kernels/_spmv.c, the
# Cython-generated C of _spmv.pyx) straight from the read-only reference tree
# into oracle/_ref/, with gcc and the flags the reference's setup.py passes
# (-O3 -fopenmp, setup.py:18-19).  The reference's own build system is NOT run.
# Output is test/baseline infrastructure only (git-ignored, travels to the GPU
# box with the snapshot).  No-op when /root/reference is absent.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src=/root/reference/pkg/src/netdos/_kernels/_spmv.c
[ -f "$src" ] || { echo "build_ref: $src absent, keeping prebuilt oracle/_ref"; exit 0; }
py=${PYTHON:-python3}
inc=$($py -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
suf=$($py -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
mkdir -p "$here/_ref"
out="$here/_ref/_spmv$suf"
if [ ! "$out" -nt "$src" ]; then
# /usr/bin/gcc: the image's default gcc cannot link -fopenmp
/usr/bin/gcc -O3 -fopenmp -fPIC -shared -I"$inc" -o "$out.tmp" "$src" -lgomp
mv "$out.tmp" "$out"
echo "build_ref: built $out"
fi
# The reference's own test modules + package sources, packed as an archive
# (never committed, never imported by the product) so tests/test_reference_suite_gpu.py
# can run them UNMODIFIED on the GPU box with netdos' moment routines rebound to
# the B200 drop-in (SURVEY.md §4 reuse plan).  Sources stay out of the tree.
tarball="$here/_ref/netdos_ref.tar.gz"
if [ ! -f "$tarball" ] || [ -n "$(find /root/reference/pkg/src/netdos /root/reference/pkg/tests -newer "$tarball" -name '*.py' -print -quit)" ]; then
  tar czf "$tarball.tmp" -C /root/reference/pkg --exclude='__pycache__' --exclude='*.so' \
      --exclude='*.c' --exclude='*.pyx' src/netdos tests
  mv "$tarball.tmp" "$tarball"
  echo "build_ref: packed $tarball"
fi
