#!/bin/bash
# Sweep the fold's grid sizes (unpipelined / pipelined, % of resident CTAs)
# on a B200 with tools/fold_sweep.py; restores the source afterwards.
# SWEEP: space-separated one_unit_pct:two_unit_pct:pipe_pct[:absmax_pct[:dequant_pct]].
set -u
cd "$(dirname "$0")/.."
SRC=paper_2510_00606_b200/csrc/kernels/weighted_reduce.cu
cp $SRC /tmp/weighted_reduce.cu.orig
for cfg in ${SWEEP:-160:100:300 100:100:200 250:300:300}; do
  set -- ${cfg//:/ }
  cp /tmp/weighted_reduce.cu.orig $SRC
  sed -i -e "s/constexpr int kFoldGrid1Pct = [0-9]*;/constexpr int kFoldGrid1Pct = $1;/" \
         -e "s/constexpr int kFoldGridPct = [0-9]*;/constexpr int kFoldGridPct = $2;/" \
         -e "s/constexpr int kFoldPipeGridPct = [0-9]*;/constexpr int kFoldPipeGridPct = $3;/" \
         -e "s/constexpr int kAbsmaxGridPct = [0-9]*;/constexpr int kAbsmaxGridPct = ${4:-100};/" \
         -e "s/constexpr int kDequantGridPct = [0-9]*;/constexpr int kDequantGridPct = ${5:-100};/" $SRC
  make -s -C paper_2510_00606_b200/csrc > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  echo "1 unit ${1}% 2 units ${2}% pipe ${3}% absmax ${4:-100}% dequant ${5:-100}%: $(timeout 200 python tools/fold_sweep.py --reps 4)"
done
cp /tmp/weighted_reduce.cu.orig $SRC
make -s -C paper_2510_00606_b200/csrc > /dev/null 2>&1
