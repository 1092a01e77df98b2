for v in 1 2 3 4; do echo "== WLB_FWD_POLY=$v"
  WLB_LIB_PATH=build_var/libP$v.so timeout 60 python tools/fwd_trace.py | tail -4
  WLB_LIB_PATH=build_var/libP$v.so timeout 60 python tools/probe_attn.py --single --iters 8
  WLB_LIB_PATH=build_var/libP$v.so timeout 60 python tools/probe_attn.py --batch 0 --iters 8
done
WLB_LIB_PATH=build_var/libP3.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
