# dQ reduction batch split A/B (dev aid)
for rep in 1 2; do for v in R8888 R8_0_12_12 R16_0_8_8 R4_4_12_12 R12_4_8_8; do
echo "$v $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --single --iters 8 | sed 's/.*| bwd/bwd/') | $(WLB_LIB_PATH=var/lib$v.so python tools/probe_attn.py --batch 1 --iters 8 | sed 's/.*| bwd/bwd/')"
done; done
