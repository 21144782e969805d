#!/bin/bash
# NOTE: the EW_REALIGN / EW_COPY_CTAS switches were removed after this sweep
# (no net gain); the script documents the experiment in profiles/r01_realign_ab_4gpu.log.
# Reshard copy A/B on 4 GPUs (bench reshard leg only): realign variant
# (EW_REALIGN=static | default select chain) x total CTAs (EW_COPY_CTAS; the
# NVLink class keeps a quarter unless EW_REMOTE_CTAS is set).
SK=e2e,inplace,replica,replay,migration,config_c,stage,philox,reduce
run() {
  timeout 300 env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 --skip $SK 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['reshard']
print('$*', r['copy_ms'], r['bottleneck_nvlink_gbs'], {k:(v['copy_ms'],v['bottleneck_nvlink_gbs']) for k,v in r['per_departure_prepared'].items()})"
}
for rep in 1 2; do
  run EW_REALIGN=select
  run EW_REALIGN=static
  run EW_REALIGN=static EW_COPY_CTAS=222 EW_REMOTE_CTAS=74
  run EW_REALIGN=static EW_COPY_CTAS=259 EW_REMOTE_CTAS=74
  run EW_REALIGN=static EW_COPY_CTAS=296 EW_REMOTE_CTAS=96
  run EW_REALIGN=select EW_COPY_CTAS=296 EW_REMOTE_CTAS=96
done
