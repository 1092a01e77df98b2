python -m pytest tests/test_cp_multi.py -m gpu -x -q 2>&1 | tail -2
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/cp_worker.py > gpurun_out/cpw2.log 2>&1; echo "cp_worker world2 rc=$?"
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n bench.py --gpus $n > gpurun_out/bench_n$n.log 2>&1; tail -1 gpurun_out/bench_n$n.log | cut -c1-400
done
