for rep in 1 2; do for v in B S N; do
echo "$v $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --single --iters 8)"
done; done
