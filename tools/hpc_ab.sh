for rep in 1 2; do for v in H2 H4 H8; do
echo "$v b1 $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --batch 1 --iters 8 | sed 's/.*median of 8: //') | d4096 $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --doc 4096 --iters 8 | sed 's/.*median of 8: //')"
done; done
