# round-end measurement set (dev aid): N=1 full line, reference arm, N=2 and N=4 (needs 4 GPUs)
python bench.py > gpurun_out/m_n1.json 2> gpurun_out/m_n1.err; tail -1 gpurun_out/m_n1.json | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err; tail -1 gpurun_out/m_ref.json | cut -c1-300
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n bench.py --gpus $n > gpurun_out/m_n$n.json 2> gpurun_out/m_n$n.err; tail -1 gpurun_out/m_n$n.json | cut -c1-300
done
