P=29600
for cfg in "4096 4 2" "8192 4 1" "8192 3 2" "16384 3 1" "16384 2 2" "4096 8 2" "8192 6 1" "2048 8 3" "4096 4 4"; do
 set -- $cfg
 P=$((P+1))
 r=$(EW_PF_SLICE=$1 EW_PF_STAGES=$2 EW_PF_CTAS_PER_SM=$3 UNITS=1 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/peer_fold_probe.py 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([round(r['rs_gbs']) for r in d['per_rank']])")
 echo "slice=$1 stages=$2 ctas=$3 -> $r"
done
