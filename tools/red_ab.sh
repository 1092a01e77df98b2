# bwd timing experiments (dev aid): B default, N no dQ writes, R dQ as TMA reduce boxes (stale data)
for rep in 1 2; do for v in B N R; do
echo "$v $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --single --iters 8 | sed 's/.*| bwd/bwd/')"
done; done
