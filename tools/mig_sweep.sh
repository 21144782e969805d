# background-transfer width vs compute stall for the layer migration leg
P=29800
for c in 32 64; do
  P=$((P+1))
  EW_MIG_CTAS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 3 --warmup 3 --skip e2e,cpu,reshard,philox,reduce,stage,replica,replay 2>/dev/null | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read())['layer_migration']; print('ctas=$c', json.dumps(r))"
done
