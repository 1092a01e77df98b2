# throughput vs uniform document length (dev aid)
for d in 256 512 1024 2048 4096 8192 32768; do
  echo "doc=$d $(python tools/probe_attn.py --doc $d --iters 6)"
done
