#!/bin/bash
# torchrun --no-python launcher: every rank under ncu with NVLink byte
# counters (device-level counters: ncu replays the whole application once per
# counter pass, on every rank in lockstep; the tool rendezvouses per pass).
#   python -m torch.distributed.run --no-python --nproc-per-node 4 ... \
#       tools/ncu_rank.sh tools/nvlink_evidence.py --reps 2
OUT=${NCU_PREFIX:-gpurun_out/ncu_nvlink}_rank${RANK}.csv
exec ncu --replay-mode application --clock-control none -k regex:"staged_copy|peer_fold" -c 16 \
  --csv --log-file "$OUT" \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum \
  python "$@"
