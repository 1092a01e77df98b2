"""Fused QKV projection + RoPE (wlb_qkv_proj_rope) vs cuBLAS GEMM + wlb_qkv_rope
at the Llama-7B / 70B-GQA projection shapes on CP ranks of a 128K micro-batch.

    python tools/proj_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import qkv_rope  # noqa: E402
from paper_2503_17924_b200.cp import project_qkv, shard_for_rank  # noqa: E402


def ev_ms(fn, reps=10):
    fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda")
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=131072)
    lengths = [d.length for d in wl.generate_synthetic_stream(spec, 0, 4)[3]]
    for name, hq, hkv, hidden in (("llama7b", 32, 32, 4096), ("llama70b-gqa", 64, 8, 8192)):
        for cp in (1, 8):
            plan = wl.build_shard_plan([lengths], cp, "per_document")
            sh = shard_for_rank(plan, 0, 0)
            tl, d = sh.gather_local.numel(), 128
            x = torch.randn(sum(lengths), hidden, device=dev, dtype=torch.bfloat16)
            xl = x[sh.gather_local.long()].contiguous()
            w = (torch.randn(hidden, (hq + 2 * hkv) * d, device=dev) / 64).to(torch.bfloat16)
            flops = 2.0 * tl * hidden * (hq + 2 * hkv) * d
            t_fused = ev_ms(lambda: project_qkv(xl, w, sh, hq, hkv, d))
            t_gather = ev_ms(lambda: project_qkv(x, w, sh, hq, hkv, d, gather=True))
            t_g4 = ev_ms(lambda: project_qkv(x, w, sh, hq, hkv, d, gather=True, gather_in_gemm=True))
            t_lib = ev_ms(lambda: qkv_rope(xl @ w, sh.tiles.positions, hq, hkv, d))
            print(json.dumps({"shape": name, "cp": cp, "rows": tl, "hidden": hidden,
                              "fused_ms": round(t_fused, 3), "fused_gather_ms": round(t_gather, 3),
                              "cublas_plus_rope_ms": round(t_lib, 3),
                              "fused_tflops": round(flops / t_fused / 1e9, 1),
                              "fused_gather_tflops": round(flops / t_gather / 1e9, 1),
                              "cublas_plus_rope_tflops": round(flops / t_lib / 1e9, 1)}), flush=True)
            del x, xl, w


if __name__ == "__main__":
    main()
