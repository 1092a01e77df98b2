run() { env $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus $2 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 N=$2', d['value'], d['imbalance'], [round(x/d['steps'],1) for x in d['rank_kernel_ms']], d['ms_per_step'])"; }
for rep in 1 2; do run WLB_XCHG_DKV=fp32 4; run WLB_XCHG_DKV=bf16 4; done
run WLB_XCHG_DKV=fp32 2; run WLB_XCHG_DKV=bf16 2
