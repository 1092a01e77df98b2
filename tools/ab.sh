# correctness + A/B of two library builds (dev aid)
WLB_LIB_PATH=build_var/libB.so timeout 150 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for n in A B; do
  echo "== $n"
  for b in 0 1; do WLB_LIB_PATH=build_var/lib$n.so timeout 60 python tools/probe_attn.py --batch $b --iters 8 | sed 's/^/  /'; done
  WLB_LIB_PATH=build_var/lib$n.so timeout 60 python tools/probe_attn.py --single --iters 8 | sed 's/^/  /'
done
