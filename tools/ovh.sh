# per-CTA fixed cost of the backward: uniform documents of growing length
for L in 128 256 512 1024 2048 4096 32768; do
  WLB_LIB_PATH=${LIB:-paper_2503_17924_b200/libwlbcp.so} timeout 60 python tools/probe_attn.py --doc $L --iters 8
done
