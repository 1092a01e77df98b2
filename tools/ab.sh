# correctness + A/B of library builds in var/ (dev aid): ab.sh B A C
T=${1:-B}
WLB_LIB_PATH=var/lib$T.so timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
for rep in 1 2; do for n in "$@"; do
  echo "== $n"
  for b in 0 1; do WLB_LIB_PATH=var/lib$n.so timeout 60 python tools/probe_attn.py --batch $b --iters 8 | sed 's/^/  /'; done
  WLB_LIB_PATH=var/lib$n.so timeout 60 python tools/probe_attn.py --single --iters 8 | sed 's/^/  /'
done; done
