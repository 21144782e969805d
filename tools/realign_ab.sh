SK=e2e,inplace,replica,replay,migration,config_c,stage,philox,reduce
for v in select static select static; do
  if [ $v = select ]; then export EW_REALIGN=select; else unset EW_REALIGN; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 --skip $SK 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['reshard']
print('$v', r['copy_ms'], r['bottleneck_nvlink_gbs'], {k:(v['copy_ms'],v['bottleneck_nvlink_gbs']) for k,v in r['per_departure_prepared'].items()})"
done
