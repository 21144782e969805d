#!/bin/bash
# Config D staged in-place reshard: slack / phase size / gather-stream sweep
# (4 GPUs).  Usage (GPU box): bash tools/inplace_sweep.sh <state_gb> ["slack phase_gb streams" ...]
S=${1:-70}
shift
CFGS=("$@")
[ ${#CFGS[@]} -eq 0 ] && CFGS=("1 2 1" "2 2 1" "4 2 1" "2 4 1" "2 1 1" "6 1 1")
P=29520
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  P=$((P+1))
  echo "# slack=$1 phase_gb=$2 gather_streams=$3"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --only-inplace \
    --inplace-state-gb $S --inplace-slack $1 --inplace-phase-gb $2 \
    --inplace-gather-streams $3 --steps 3 --warmup 3 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])['inplace']; print(json.dumps({k: d[k] for k in ('slack','phases','gather_streams','staging_buffers','stage_bytes','copy_ms','bottleneck_nvlink_gbs','verified_on_arrival','verified_by_reread','peak_hbm_allocated_gb')}))"
done
