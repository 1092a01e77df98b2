for rep in 1 2; do for v in P2 P4 P8; do
echo "$v d512 $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --doc 512 --iters 8 | sed 's/.*median of 8: //; s/(min.*//') | d2048 $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --doc 2048 --iters 8 | sed 's/.*median of 8: //; s/(min.*//') | b3 $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --batch 3 --iters 8 | sed 's/.*median of 8: //; s/(min.*//')"
done; done
