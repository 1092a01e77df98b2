python bench.py --shape llama70b-gqa --no-cpu-baseline > gpurun_out/g_n1.json 2> gpurun_out/g_n1.err; tail -1 gpurun_out/g_n1.json | cut -c1-200
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n --shape llama70b-gqa > gpurun_out/g_n$n.json 2> gpurun_out/g_n$n.err; tail -1 gpurun_out/g_n$n.json | cut -c1-200
done
