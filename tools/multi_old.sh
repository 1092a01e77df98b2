for rep in 1 2; do
( cd var/old && python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29657 bench.py --gpus 4 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('OLD', d['value'], d['imbalance'], d['rank_kernel_ms'], d['ms_per_step'], d['clocks']['sm_mhz'])" )
WLB_LIB_PATH=var/libB.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29658 bench.py --gpus 4 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('NEW', d['value'], d['imbalance'], d['rank_kernel_ms'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
