#!/usr/bin/env bash
# Round 2 GPU call W: gather roofline by segment size (tools/exp/gather_bw.cu)
# and the default bench line on the final build (traffic.json keyed to it).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 ./tools/exp/gather_bw > gpurun_out/r2_w_gather_bw.log 2>&1
echo "rc=$?" >> gpurun_out/r2_w_gather_bw.log
( time timeout 1500 python bench.py ) > gpurun_out/r2_w_bench.log 2>&1
echo "rc=$?" >> gpurun_out/r2_w_bench.log
