for v in 0 1; do echo "== WLB_FWD_TURNS=$v"
  WLB_LIB_PATH=build_var/libR$v.so timeout 60 python tools/fwd_trace.py | tail -5
  WLB_LIB_PATH=build_var/libR$v.so timeout 60 python tools/probe_attn.py --single --iters 8
  WLB_LIB_PATH=build_var/libR$v.so timeout 60 python tools/probe_attn.py --batch 0 --iters 8
  WLB_LIB_PATH=build_var/libR$v.so timeout 60 python tools/probe_attn.py --batch 1 --iters 8
done
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
