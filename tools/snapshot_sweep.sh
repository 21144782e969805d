#!/bin/bash
# Sweep the register-staged snapshot kernel's shape (threads per CTA, loads
# in flight per lane, register cap) on a B200: rewrite the constants in
# snapshot.cu, rebuild the library, time with tools/snapshot_time.py.
# Restores the source afterwards.  Usage: bash tools/snapshot_sweep.sh
set -u
cd "$(dirname "$0")/.."
SRC=paper_2510_00606_b200/csrc/kernels/snapshot.cu
cp $SRC /tmp/snapshot.cu.orig
# SWEEP: space-separated threads:unroll:min_blocks[:grid_pct[:stagger]] tuples
for cfg in ${SWEEP:-128:4:8 128:4:6 128:4:4 128:2:12 128:2:8 256:4:4 256:4:3 256:2:6 64:4:16}; do
  set -- ${cfg//:/ }
  cp /tmp/snapshot.cu.orig $SRC
  sed -i -e "s/constexpr int kWarpRowThreads = [0-9]*;/constexpr int kWarpRowThreads = $1;/" \
         -e "s/constexpr int kWarpRowUnroll = [0-9]*;/constexpr int kWarpRowUnroll = $2;/" \
         -e "s/constexpr int kWarpRowMinBlocks = [0-9]*;/constexpr int kWarpRowMinBlocks = $3;/" \
         -e "s/constexpr int kWarpRowGridPct = [0-9]*;/constexpr int kWarpRowGridPct = ${4:-100};/" \
         -e "s/constexpr int kWarpRowStagger = [0-9]*;/constexpr int kWarpRowStagger = ${5:-5};/" $SRC
  make -s -C paper_2510_00606_b200/csrc > /dev/null 2>&1 || { echo "{\"tag\": \"$1 $2 $3\", \"build\": \"failed\"}"; continue; }
  regs=$(cuobjdump -res-usage paper_2510_00606_b200/libelaskit_b200.so 2>/dev/null | grep -A1 'warp_row_kernelILNS0_4ModeE0' | grep -oE 'REG:[0-9]+ STACK:[0-9]+' | head -1)
  timeout 300 python tools/snapshot_time.py --tag "T$1 U$2 minB$3 grid${4:-100}% stagger${5:-5} $regs"
done
cp /tmp/snapshot.cu.orig $SRC
make -s -C paper_2510_00606_b200/csrc > /dev/null 2>&1
