# A/B of the AdamW replay kernels at N=4 (bench.py replay leg only)
P=29700
for cfg in "0 8 2" "0 8 1" "0 8 3" "0 8 4" "0 4 4" "0 16 1"; do  # staged flag column kept for old logs; ignored now
  set -- $cfg; P=$((P+1))
  EW_ADAM_STAGED=$1 EW_ADAM_CTAS_PER_SM=$2 EW_ADAM_DEPTH=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 3 --warmup 3 --skip e2e,cpu,reshard,philox,reduce,stage,replica 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['replay']; print('staged=$1 ctas=$2 depth=$3', r['owner_step_ms'], r['owner_step_hbm_gbs'], r['holder_replay_ms'], r['nvlink_gbs'], r['replica_verified_every_step'])"
done
