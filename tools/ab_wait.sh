for v in 0 1 2; do echo "== WLB_MMA_WAIT=$v"
  WLB_LIB_PATH=build_var/libT$v.so timeout 60 python tools/fwd_trace.py | tail -4
  WLB_LIB_PATH=build_var/libT$v.so timeout 60 python tools/probe_attn.py --single --iters 8
  WLB_LIB_PATH=build_var/libT$v.so timeout 60 python tools/probe_attn.py --batch 0 --iters 8
done
