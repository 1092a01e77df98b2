# round-end measurement set (dev aid, 4 GPUs)
python -m pytest tests -m gpu -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/measure_all.sh
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29674 bench.py --gpus 4 --shape llama70b-gqa > gpurun_out/g_n4.json 2> gpurun_out/g_n4.err; tail -1 gpurun_out/g_n4.json | cut -c1-200
