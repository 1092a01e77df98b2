for rep in 1 2; do for p in 0 1; do
echo "pairs=$p $(python tools/probe_attn.py --single --iters 8 --pairs $p) | $(python tools/probe_attn.py --batch 1 --iters 8 --pairs $p | sed 's/.*bwd/bwd/') | $(python tools/probe_attn.py --doc 8192 --iters 8 --pairs $p | sed 's/.*bwd/bwd/')"
done; done
