# N=4 bench A/B of library builds (dev aid): multi_ab.sh A B ...
for rep in 1 2; do for v in "$@"; do
WLB_LIB_PATH=var/lib$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 4 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['imbalance'], [round(x/d['steps'],1) for x in d['rank_kernel_ms']], d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
