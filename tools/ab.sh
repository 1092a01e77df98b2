for rep in 1 2; do for n in A B; do
  echo "== $n"
  for b in 0 1; do WLB_LIB_PATH=build_var/lib$n.so timeout 60 python tools/probe_attn.py --batch $b --iters 8 | sed 's/^/  /'; done
  WLB_LIB_PATH=build_var/lib$n.so timeout 60 python tools/probe_attn.py --single --iters 8 | sed 's/^/  /'
done; done
