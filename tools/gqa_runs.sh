python bench.py --shape llama70b-gqa --no-cpu-baseline > gpurun_out/g_n1.json 2> gpurun_out/g_n1.err; tail -1 gpurun_out/g_n1.json | cut -c1-120
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 --shape llama70b-gqa > gpurun_out/g_n2.json 2> gpurun_out/g_n2.err; tail -1 gpurun_out/g_n2.json | cut -c1-120
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29673 tests/cp_worker.py > gpurun_out/cpw2.log 2>&1; echo "cp_worker world2 rc=$?"
