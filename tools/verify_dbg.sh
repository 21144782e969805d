# A/B of verification-on-arrival settings for the N=4 reshard leg (remote CTA count)
P=29700
for c in 74 86 98; do P=$((P+1))
EW_REMOTE_CTAS=$c python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --skip e2e,cpu,philox,reduce,stage,replica,replay,migration 2>/dev/null | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read())[\"reshard\"]; print('remote_ctas=$c', r[\"mttr_ms\"][\"copy\"], r[\"copy_without_verification_ms\"], r[\"verified_by_checksums\"])"
done
