# A/B forward variants on the long single doc and the 6-doc batch
for n in A B C D E; do
  echo "== $n"; WLB_LIB_PATH=build_var/lib$n.so timeout 60 python tools/probe_attn.py --single --iters 8 | sed 's/^/  /'
  WLB_LIB_PATH=build_var/lib$n.so timeout 60 python tools/probe_attn.py --batch 1 --iters 8 | sed 's/^/  /'
done
