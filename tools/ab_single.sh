# quick A/B on the long single document and the 6-doc batch (dev aid): ab_single.sh B R1 ...
for rep in 1 2; do for n in "$@"; do
  echo "== $n $(WLB_LIB_PATH=var/lib$n.so timeout 60 python tools/probe_attn.py --single --iters 8) | $(WLB_LIB_PATH=var/lib$n.so timeout 60 python tools/probe_attn.py --batch 1 --iters 8 | sed 's/.*bwd/bwd/')"
done; done
