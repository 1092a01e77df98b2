# backward A/B of library builds (dev aid): bwd_ab.sh A B ...
for rep in 1 2 3; do for v in "$@"; do
echo "$v $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --single --iters 8 | sed 's/.*| bwd/bwd/; s/(min.*//') | $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --batch 1 --iters 8 | sed 's/.*| bwd/bwd/; s/(min.*//')"
done; done
