#!/bin/bash
# torchrun --no-python launcher: profile ONE rank (NCU_RANK, default 1) of a
# multi-process run with ncu's NVLink byte counters; the other ranks run
# plainly and wait at host barriers while the profiled kernels replay.
#   python -m torch.distributed.run --no-python --nproc-per-node 4 ... \
#       tools/ncu_rank.sh tools/nvlink_evidence.py --reps 2
OUT=${NCU_OUT:-gpurun_out/ncu_nvlink_rank${NCU_RANK:-1}.csv}
if [ "$RANK" = "${NCU_RANK:-1}" ]; then
  exec ncu --replay-mode kernel --clock-control none -k regex:"staged_copy|peer_fold" -c 16 --csv --log-file "$OUT" \
    --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum \
    python "$@"
else
  exec python "$@"
fi
