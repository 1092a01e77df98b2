// GPU CP shard builder + adaptive selector (north-star items 1 and 4).
//
// Replaces, bit-exactly, the reference's host loops:
//   per_sequence_shard  sharding.py:86-110   (per-(worker, doc) overlap walk)
//   per_document_shard  sharding.py:113-141  (per-token remainder loop)
//   _canonical          sharding.py:63-74    (sort + merge)
//   worker_attention_latency / strategy_latencies / adaptive_select
//                       sharding.py:151-188, _compiled.pyx:30-47
//
// Instead of building raw spans and sorting, each (worker, doc) pair evaluates
// the closed form of its canonical ranges directly (at most 4 per-document,
// at most 2 per-sequence), so the whole micro-batch is embarrassingly
// parallel after one prefix scan of document starts and remainder counts:
//
//   per-document: d = L/2cp, R = L mod 2cp, c0 = (sum_{q<p} R_q) mod cp
//     worker w owns [w d,(w+1) d) and [(2cp-1-w) d,(2cp-w) d) (merged when
//     w = cp-1), plus tail tokens 2cp d + k for k in {k1, k1+cp} < R,
//     k1 = (w - c0) mod cp; the first tail token merges into worker 0's last
//     chunk when k1 = 0.
//   per-sequence: C = T/2cp, worker w owns global chunks w and 2cp-1-w,
//     clipped to each document (merged at the middle when w = cp-1).
//
// One CTA per micro-batch: config 5 (64 micro-batches per step) is one launch.
#include "common.cuh"

namespace wlb {

struct Seg {
  int s, e;
};

// Canonical ranges of worker w inside document p, per-document strategy.
__device__ __forceinline__ int per_doc_ranges(long long L, long long cursor, int cp, int w,
                                              Seg* out) {
  const long long two = 2LL * cp;
  const long long d = L / two, R = L % two, ts = two * d;
  const int c0 = (int)(cursor % cp);
  int n = 0;
  if (d > 0) {
    if (w == cp - 1) {
      out[n++] = {(int)(w * d), (int)((w + 2) * d)};
    } else {
      out[n++] = {(int)(w * d), (int)((w + 1) * d)};
      out[n++] = {(int)((two - 1 - w) * d), (int)((two - w) * d)};
    }
  }
  int k1 = ((w - c0) % cp + cp) % cp;
  for (long long k = k1; k < R; k += cp) {
    int t = (int)(ts + k);
    if (n && out[n - 1].e == t) out[n - 1].e = t + 1;
    else out[n++] = {t, t + 1};
  }
  return n;
}

// Canonical ranges of worker w inside document p (global span [A, B)),
// per-sequence strategy with chunk size C.
__device__ __forceinline__ int per_seq_ranges(long long A, long long B, long long C, int cp,
                                              int w, Seg* out) {
  int n = 0;
  if (C == 0) return 0;
  const long long chunks[2] = {(long long)w, 2LL * cp - 1 - w};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    long long lo = chunks[i] * C, hi = lo + C;
    long long a = lo > A ? lo : A, b = hi < B ? hi : B;
    if (a < b) {
      int s = (int)(a - A), e = (int)(b - A);
      if (n && out[n - 1].e == s) out[n - 1].e = e;
      else out[n++] = {s, e};
    }
  }
  return n;
}

__device__ __forceinline__ double range_latency(long long q, long long kv, long long tile,
                                                const long long* cq, const double* cv,
                                                int ncurve, double op_scale) {
  int j = ncurve - 1;
  while (j > 0 && cq[j] > q) --j;
  long long padded = ((q + tile - 1) / tile) * tile;
  // op_scale * (double)(padded*kv) / cv[j], rounded exactly as the reference.
  return __ddiv_rn(__dmul_rn(op_scale, (double)(padded * kv)), cv[j]);
}

// ---------------------------------------------------------------------------
// Measured-latency selector (north-star item 4; PAPER.md:425-429 selects with
// profiled kernel latency).  The reference-form CostProfile charges each
// canonical range as a dense q x kv rectangle (workload.py:239-255) and cannot
// see what the B200 kernels actually run.  This model prices the work lists
// themselves, per (strategy, rank), from the canonical ranges:
//   forward : back-aligned 128-row query tiles of each (rank, document)
//             row-set, paired from the end (wlb_attn_tiles); a tile costs one
//             step per 128-key KV tile below its last row's position
//   backward: 128-key KV tiles of each row-set up to its last position
//             (bwd_kv_tiles_kernel); a KV tile costs one step per 64-query
//             (v2) or 128-query (v3) tile of the rows that can see it
// Integer features per (strategy, rank), kFeat of them:
enum { kF_ITEMS = 0, kF_STEPS, kF_MAX, kB_ITEMS, kB_Q64, kB_Q128, kB_MAX64, kB_MAX128, kFeat };
// and model[WLB_TILE_MODEL_LEN] (seconds): per direction, with the even
// spread S and the largest item M,
//   Sf = (fi*F_ITEMS + fs*F_STEPS) * Hq / SMs,   Mf = fi + fs*F_MAX
//   Sb = (bi*B_ITEMS*Hkv + bs*B_Q*Hq) / SMs,     Mb = bi + bs*B_MAX*(Hq/Hkv)
//   t = max(Sf, Mf) + gf*min(Sf, Mf) + max(Sb, Mb) + gb*min(Sb, Mb) + c0
// (g: the list-scheduling tail the largest item adds; tilemodel.py),
// bi / B_Q / B_MAX / bs of the backward kernel the library will pick (v3 when
// the rank's rows per document reach v3_min_rows and D = 128).
constexpr int kMaxModelCp = 64;

__device__ __forceinline__ int rowset_pos(const Seg* r, int n, int i) {
  for (int k = 0; k < n; ++k) {
    const int len = r[k].e - r[k].s;
    if (i < len) return r[k].s + i;
    i -= len;
  }
  return r[n - 1].e - 1;
}

__device__ void tile_model_select(int b, int nd, const long long* L, const long long* dstart,
                                  const long long* cursor, long long C, int cp, int policy,
                                  const double* model, long long* features, double* rank_latency,
                                  int* choice, int* chosen_s) {
  __shared__ unsigned long long feat[2][kMaxModelCp][kFeat];
  for (int i = threadIdx.x; i < 2 * kMaxModelCp * kFeat; i += blockDim.x)
    (&feat[0][0][0])[i] = 0;
  __syncthreads();
  for (long long it = threadIdx.x; it < 2LL * cp * nd; it += blockDim.x) {
    const int strat = (int)(it / ((long long)cp * nd));
    const int w = (int)((it / nd) % cp), p = (int)(it % nd);
    Seg r[4];
    const int n = strat ? per_doc_ranges(L[p], cursor[p], cp, w, r)
                        : per_seq_ranges(dstart[p], dstart[p + 1], C, cp, w, r);
    if (n == 0) continue;
    int R = 0;
    for (int k = 0; k < n; ++k) R += r[k].e - r[k].s;
    // forward: tiles from the end, paired (X = later, Y = earlier)
    const int nt = (R + 127) / 128;
    unsigned long long steps = 0, fmax = 0;
    for (int t = 0; t < nt; t += 2) {
      const unsigned long long kx = (rowset_pos(r, n, R - 1 - 128 * t) + 128) / 128;
      const unsigned long long ky = t + 1 < nt ? (rowset_pos(r, n, R - 1 - 128 * (t + 1)) + 128) / 128 : 0;
      steps += kx + ky;
      fmax = max(fmax, kx + ky);
    }
    // backward: KV tiles below the last position, rows with position >= k0
    const int nkv = (r[n - 1].e - 1 + 128) / 128;
    unsigned long long q64 = 0, q128 = 0, m64 = 0, m128 = 0;
    for (int t = 0; t < nkv; ++t) {
      const int k0 = 128 * t;
      int cnt = 0;
      for (int k = 0; k < n; ++k) cnt += max(0, r[k].e - max(r[k].s, k0));
      const unsigned long long a = (cnt + 63) / 64, c = (cnt + 127) / 128;
      q64 += a;
      q128 += c;
      m64 = max(m64, a);
      m128 = max(m128, c);
    }
    unsigned long long* f = feat[strat][w];
    atomicAdd(&f[kF_ITEMS], (unsigned long long)((nt + 1) / 2));
    atomicAdd(&f[kF_STEPS], steps);
    atomicMax(&f[kF_MAX], fmax);
    atomicAdd(&f[kB_ITEMS], (unsigned long long)nkv);
    atomicAdd(&f[kB_Q64], q64);
    atomicAdd(&f[kB_Q128], q128);
    atomicMax(&f[kB_MAX64], m64);
    atomicMax(&f[kB_MAX128], m128);
  }
  __syncthreads();
  if (features)
    for (int i = threadIdx.x; i < 2 * cp * kFeat; i += blockDim.x)
      features[(long long)b * 2 * cp * kFeat + i] = (long long)(&feat[0][0][0])[(i / (cp * kFeat)) * kMaxModelCp * kFeat + i % (cp * kFeat)];
  if (threadIdx.x < 2 * cp) {
    const int strat = threadIdx.x / cp, w = threadIdx.x % cp;
    const unsigned long long* f = feat[strat][w];
    const double sms = model[0], hq = model[1], hkv = model[2];
    const double fi = model[3], fs = model[4], bi = model[5], bs64 = model[6], bs128 = model[7];
    const double v3_rows = model[8], c0 = model[9], d128 = model[10], bi128 = model[11];
    const double gf = model[12], gb = model[13];
    const long long T = dstart[nd];
    const bool v3 = d128 != 0.0 && (double)(T / cp) >= v3_rows * (double)(nd > 0 ? nd : 1);
    const double bq = (double)(v3 ? f[kB_Q128] : f[kB_Q64]);
    const double bm = (double)(v3 ? f[kB_MAX128] : f[kB_MAX64]);
    const double bs = v3 ? bs128 : bs64, bi_k = v3 ? bi128 : bi;
    const double sf = (fi * (double)f[kF_ITEMS] + fs * (double)f[kF_STEPS]) * hq / sms;
    const double mf = fi + fs * (double)f[kF_MAX];
    const double sb = (bi_k * (double)f[kB_ITEMS] * hkv + bs * bq * hq) / sms;
    const double mb = bi_k + bs * bm * (hq / hkv);
    const double tf = fmax(sf, mf) + gf * fmin(sf, mf);
    const double tb = fmax(sb, mb) + gb * fmin(sb, mb);
    rank_latency[((long long)b * 2 + strat) * cp + w] = tf + tb + c0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = policy;
    if (policy == WLB_POLICY_MEASURED) {
      double g[2];
      for (int s = 0; s < 2; ++s) {
        g[s] = 0.0;
        for (int w = 0; w < cp; ++w) g[s] = fmax(g[s], rank_latency[((long long)b * 2 + s) * cp + w]);
      }
      c = g[0] <= g[1] ? WLB_STRATEGY_PER_SEQUENCE : WLB_STRATEGY_PER_DOCUMENT;
    }
    *chosen_s = c;
    choice[b] = c;
  }
}

constexpr int kPlanThreads = 512;
constexpr int kSmemDocs = 12000;   // documents whose starts + cursors fit shared memory (188 KB)

__global__ void __launch_bounds__(kPlanThreads)
shard_plan_kernel(const int* __restrict__ mb_doc_off, const long long* __restrict__ doc_len,
                  const long long* __restrict__ mb_tok_off, int cp, int policy, long long tile,
                  const long long* __restrict__ curve_q, const double* __restrict__ curve_v,
                  int n_curve, double op_scale, int max_segs, int max_docs,
                  int* __restrict__ choice, double* __restrict__ rank_latency,
                  long long* __restrict__ rank_pairs, int* __restrict__ seg_count,
                  int* __restrict__ segs, int* __restrict__ rowset_off,
                  int* __restrict__ gather_index, int* __restrict__ positions,
                  long long* __restrict__ gscratch, const double* __restrict__ model,
                  long long* __restrict__ features) {
  extern __shared__ long long smem_ll[];
  __shared__ long long warp_tot[kPlanThreads / 32 + 1];
  __shared__ long long total_s;
  __shared__ int chosen_s;

  const int b = blockIdx.x;
  // document starts [max_docs+1] and remainder cursor [max_docs]: shared
  // memory, or this micro-batch's slice of a global scratch when they do not
  // fit (more than kSmemDocs documents)
  long long* dstart = gscratch ? gscratch + (size_t)b * (2 * (size_t)max_docs + 1) : smem_ll;
  long long* cursor = dstart + max_docs + 1;
  const int d0 = mb_doc_off[b];
  const int nd = mb_doc_off[b + 1] - d0;
  const long long* L = doc_len + d0;
  const int two = 2 * cp;

  // -- 1. prefix scans: document starts and remainder cursor --------------------
  long long carry_len = 0, carry_rem = 0;
  for (int base = 0; base < nd; base += blockDim.x) {
    int p = base + threadIdx.x;
    long long len = p < nd ? L[p] : 0;
    long long tot_len, tot_rem;
    long long ex_len = block_exclusive_scan(len, warp_tot, &tot_len);
    long long ex_rem = block_exclusive_scan(len % two, warp_tot, &tot_rem);
    if (p < nd) {
      dstart[p] = carry_len + ex_len;
      cursor[p] = carry_rem + ex_rem;
    }
    carry_len += tot_len;
    carry_rem += tot_rem;
  }
  if (threadIdx.x == 0) {
    dstart[nd] = carry_len;
    total_s = carry_len;
  }
  __syncthreads();
  const long long T = total_s;
  if (T % two != 0) {
    if (threadIdx.x == 0) choice[b] = -1;
    return;
  }
  const long long C = T / two;

  // -- 2. canonical ranges of both strategies, all workers ---------------------
  for (int strat = 0; strat < 2; ++strat) {
    for (int w = 0; w < cp; ++w) {
      int* out = segs + ((((long long)b * 2 + strat) * cp + w) * max_segs) * 3;
      long long carry = 0;
      for (int base = 0; base < nd; base += blockDim.x) {
        int p = base + threadIdx.x;
        Seg r[4];
        int n = 0;
        if (p < nd)
          n = strat ? per_doc_ranges(L[p], cursor[p], cp, w, r)
                    : per_seq_ranges(dstart[p], dstart[p + 1], C, cp, w, r);
        long long tot;
        long long off = carry + block_exclusive_scan(n, warp_tot, &tot);
        for (int i = 0; i < n; ++i) {
          if (off + i < max_segs) {
            out[(off + i) * 3 + 0] = p;
            out[(off + i) * 3 + 1] = r[i].s;
            out[(off + i) * 3 + 2] = r[i].e;
          }
        }
        carry += tot;
      }
      if (threadIdx.x == 0) seg_count[((long long)b * 2 + strat) * cp + w] = (int)carry;
    }
  }
  __syncthreads();
  __threadfence_block();

  if (model) {
    // -- 3'. measured policy: price both strategies from the work lists the
    //        attention kernels will run, with B200-calibrated per-tile costs
    tile_model_select(b, nd, L, dstart, cursor, C, cp, policy, model, features, rank_latency,
                      choice, &chosen_s);
  } else {
  // -- 3. per-worker model latency (sequential, canonical order: bit-exact) ----
  if (threadIdx.x < 2 * cp) {
    const int strat = threadIdx.x / cp, w = threadIdx.x % cp;
    const int n = seg_count[((long long)b * 2 + strat) * cp + w];
    const int* in = segs + ((((long long)b * 2 + strat) * cp + w) * max_segs) * 3;
    double tot = 0.0;
    for (int i = 0; i < n && i < max_segs; ++i) {
      long long s = in[i * 3 + 1], e = in[i * 3 + 2];
      tot = __dadd_rn(tot, range_latency(e - s, e, tile, curve_q, curve_v, n_curve, op_scale));
    }
    rank_latency[((long long)b * 2 + strat) * cp + w] = tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = policy;
    if (policy == WLB_POLICY_ADAPTIVE) {
      double g[2];
      for (int s = 0; s < 2; ++s) {
        g[s] = 0.0;
        for (int w = 0; w < cp; ++w) g[s] = fmax(g[s], rank_latency[((long long)b * 2 + s) * cp + w]);
      }
      c = g[0] <= g[1] ? WLB_STRATEGY_PER_SEQUENCE : WLB_STRATEGY_PER_DOCUMENT;
    }
    chosen_s = c;
    choice[b] = c;
  }
  }
  __syncthreads();
  const int strat = chosen_s;

  // -- 4. chosen strategy: pairs, row-set offsets, token layout -----------------
  const long long tok0 = mb_tok_off ? mb_tok_off[b] : 0;
  const long long rows_per_rank = T / cp;
  for (int w = 0; w < cp; ++w) {
    const int n = seg_count[((long long)b * 2 + strat) * cp + w];
    const int* in = segs + ((((long long)b * 2 + strat) * cp + w) * max_segs) * 3;
    // pairs
    long long pr = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      long long s = in[i * 3 + 1], e = in[i * 3 + 2];
      pr += (e * (e + 1) - s * (s + 1)) / 2;
    }
    long long tot;
    block_exclusive_scan(pr, warp_tot, &tot);
    if (threadIdx.x == 0) rank_pairs[(long long)b * cp + w] = tot;
    // row-set offsets: tokens of (w, p) via the closed form again
    int* ro = rowset_off ? rowset_off + ((long long)b * cp + w) * (max_docs + 1) : nullptr;
    long long carry = 0;
    for (int base = 0; base < nd; base += blockDim.x) {
      int p = base + threadIdx.x;
      Seg r[4];
      int k = 0;
      if (p < nd)
        k = strat ? per_doc_ranges(L[p], cursor[p], cp, w, r)
                  : per_seq_ranges(dstart[p], dstart[p + 1], C, cp, w, r);
      long long cnt = 0;
      for (int i = 0; i < k; ++i) cnt += r[i].e - r[i].s;
      long long t2;
      long long ex = block_exclusive_scan(cnt, warp_tot, &t2);
      if (ro && p < nd) ro[p] = (int)(carry + ex);
      carry += t2;
    }
    if (ro && threadIdx.x == 0) ro[nd] = (int)carry;
    // token layout: local rows = concatenation of canonical ranges
    if (gather_index || positions) {
      long long row = 0;
      for (int i = 0; i < n; ++i) {
        const int p = in[i * 3 + 0], s = in[i * 3 + 1], e = in[i * 3 + 2];
        const long long dst = tok0 + w * rows_per_rank + row;
        for (int t = threadIdx.x; t < e - s; t += blockDim.x) {
          if (gather_index) gather_index[dst + t] = (int)(dstart[p] + s + t);
          if (positions) positions[dst + t] = s + t;
        }
        row += e - s;
      }
    }
  }
}

__global__ void kernel_latency_sum_kernel(const long long* q, const long long* kv, long long n,
                                          long long tile, const long long* cq, const double* cv,
                                          int ncurve, double op_scale, double* out) {
  // Sequential by construction: fp64 addition order must equal the reference's.
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double tot = 0.0;
  for (long long i = 0; i < n; ++i)
    if (q[i] != 0) tot = __dadd_rn(tot, range_latency(q[i], kv[i], tile, cq, cv, ncurve, op_scale));
  out[0] = tot;
}

// ---------------------------------------------------------------------------
// Attention work list.  Row-set (rank, doc) rows are sorted by in-document
// position; a query tile's cost is its KV extent (last row position + 1).
// Because the optimal cost f(i) of tiling the first i rows is non-decreasing
// in i, f(i) = f(i - BM) + cost(last tile): back-aligned tiling (partial tile
// first) is optimal.  Adjacent tiles of a row-set are then paired from the
// end -- a pair shares every K/V tile of the shorter member -- and the pairs
// are counting-sorted by descending KV extent so the persistent-style grid
// schedules longest-first (LPT).
//   item[2i]   = {rowX0, nrowsX, kv_begin, kv_endX}   X = later tile (longer KV)
//   item[2i+1] = {rowY0, nrowsY, kv_endY, 0}          Y = earlier tile, nrowsY may be 0
constexpr int kTileThreads = 1024;
constexpr int kTileBins = 2048;

__global__ void __launch_bounds__(kTileThreads)
attn_tiles_kernel(int nd, const int* __restrict__ rowset_off, const int* __restrict__ positions,
                  const int* __restrict__ doc_start, int bm, int max_items, int4* __restrict__ items,
                  int* __restrict__ n_items, int4* __restrict__ scratch) {
  __shared__ long long warp_tot[kTileThreads / 32 + 1];
  __shared__ int hist[kTileBins];
  __shared__ int kv_shift_s;
  // pass 1: pair count per doc -> offsets; emit unsorted pairs into scratch
  long long carry = 0;
  for (int base = 0; base < nd; base += blockDim.x) {
    int p = base + threadIdx.x;
    int rows = p < nd ? rowset_off[p + 1] - rowset_off[p] : 0;
    int nt = (rows + bm - 1) / bm;
    int npairs = (nt + 1) / 2;
    long long tot;
    long long off = carry + block_exclusive_scan(npairs, warp_tot, &tot);
    if (p < nd) {
      const int r0 = rowset_off[p], r1 = rowset_off[p + 1];
      for (int k = 0; k < npairs; ++k) {
        // tiles counted from the end: X = tile nt-1-2k, Y = tile nt-2-2k (if any)
        const int endX = r1 - 2 * k * bm;
        const int begX = endX - bm > r0 ? endX - bm : r0;
        const int kvX = doc_start[p] + positions[endX - 1] + 1;
        int begY = begX, nY = 0, kvY = 0;
        if (begX > r0) {
          const int endY = begX;
          begY = endY - bm > r0 ? endY - bm : r0;
          nY = endY - begY;
          kvY = doc_start[p] + positions[endY - 1] + 1;
        }
        if (off + k < max_items) {
          scratch[2 * (off + k)] = make_int4(begX, endX - begX, doc_start[p], kvX);
          scratch[2 * (off + k) + 1] = make_int4(begY, nY, kvY, 0);
        }
      }
    }
    carry += tot;
  }
  const int total = carry < max_items ? (int)carry : max_items;
  // pass 2: counting sort by descending KV extent (in 128-key blocks)
  int max_ext = 0;
  for (int i = threadIdx.x; i < total; i += blockDim.x)
    max_ext = max(max_ext, (scratch[2 * i].w - scratch[2 * i].z + 127) >> 7);
  for (int o = 16; o; o >>= 1) max_ext = max(max_ext, __shfl_xor_sync(0xffffffffu, max_ext, o));
  if (threadIdx.x == 0) kv_shift_s = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicMax(&kv_shift_s, max_ext);
  __syncthreads();
  int shift = 0;
  while ((kv_shift_s >> shift) >= kTileBins) ++shift;
  for (int i = threadIdx.x; i < kTileBins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    int key = kTileBins - 1 - (((scratch[2 * i].w - scratch[2 * i].z + 127) >> 7) >> shift);
    atomicAdd(&hist[key], 1);
  }
  __syncthreads();
  long long a0 = hist[2 * threadIdx.x], a1 = hist[2 * threadIdx.x + 1], tot;
  long long ex = block_exclusive_scan(a0 + a1, warp_tot, &tot);
  hist[2 * threadIdx.x] = (int)ex;
  hist[2 * threadIdx.x + 1] = (int)(ex + a0);
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    int key = kTileBins - 1 - (((scratch[2 * i].w - scratch[2 * i].z + 127) >> 7) >> shift);
    int slot = atomicAdd(&hist[key], 1);
    items[2 * slot] = scratch[2 * i];
    items[2 * slot + 1] = scratch[2 * i + 1];
  }
  if (threadIdx.x == 0) n_items[0] = total;
}

}  // namespace wlb

using namespace wlb;

static int launch_plan(int32_t n_mb, const int32_t* mb_doc_off, const int64_t* doc_len,
                       const int64_t* mb_tok_off, int32_t cp, int32_t policy, int64_t tile,
                       const int64_t* curve_q, const double* curve_v, int32_t n_curve,
                       double op_scale, int32_t max_segs, int32_t max_docs, int32_t* choice,
                       double* rank_latency, int64_t* rank_pairs, int32_t* seg_count,
                       int32_t* segs, int32_t* rowset_off, int32_t* gather_index,
                       int32_t* positions, const double* model, int64_t* features,
                       cudaStream_t stream) {
  WLB_REQUIRE(max_docs >= 1, "max_docs out of range");
  WLB_REQUIRE(max_segs >= 4 * (int64_t)max_docs + 2, "max_segs must be >= 4*max_docs+2");
  if (n_mb <= 0) return WLB_OK;
  const size_t per_mb = sizeof(long long) * (2 * (size_t)max_docs + 1);
  long long* gscratch = nullptr;
  size_t smem = per_mb;
  // the measured policy's per-(strategy, rank) features take 8 KB of static smem
  const int smem_docs = model ? kSmemDocs - 512 : kSmemDocs;
  if (max_docs > smem_docs) {
    // stream-ordered global scratch (freed after the launch, on the same stream)
    WLB_CUDA_TRY(cudaMallocAsync((void**)&gscratch, per_mb * (size_t)n_mb, stream));
    smem = 0;
  } else if (smem > 48 * 1024) {
    WLB_SMEM_ATTR(shard_plan_kernel, (int)smem);
  }
  shard_plan_kernel<<<n_mb, kPlanThreads, smem, stream>>>(
      mb_doc_off, (const long long*)doc_len, (const long long*)mb_tok_off, cp, policy, tile,
      (const long long*)curve_q, curve_v, n_curve, op_scale, max_segs, max_docs, choice,
      rank_latency, (long long*)rank_pairs, seg_count, segs, rowset_off, gather_index, positions,
      gscratch, model, (long long*)features);
  WLB_LAUNCH_CHECK();
  if (gscratch) WLB_CUDA_TRY(cudaFreeAsync(gscratch, stream));
  return WLB_OK;
}

extern "C" int wlb_shard_plan(int32_t n_mb, const int32_t* mb_doc_off, const int64_t* doc_len,
                              const int64_t* mb_tok_off, int32_t cp, int32_t policy, int64_t tile,
                              const int64_t* curve_q, const double* curve_v, int32_t n_curve,
                              double op_scale, int32_t max_segs, int32_t max_docs, int32_t* choice,
                              double* rank_latency, int64_t* rank_pairs, int32_t* seg_count,
                              int32_t* segs, int32_t* rowset_off, int32_t* gather_index,
                              int32_t* positions, void* stream) {
  WLB_REQUIRE(cp >= 1, "cp must be >= 1");
  WLB_REQUIRE(policy >= 0 && policy <= 2, "unknown policy %d", policy);
  WLB_REQUIRE(n_curve >= 1 && tile >= 1, "bad cost profile");
  return launch_plan(n_mb, mb_doc_off, doc_len, mb_tok_off, cp, policy, tile, curve_q, curve_v,
                     n_curve, op_scale, max_segs, max_docs, choice, rank_latency, rank_pairs,
                     seg_count, segs, rowset_off, gather_index, positions, nullptr, nullptr,
                     (cudaStream_t)stream);
}

extern "C" int wlb_shard_plan_measured(int32_t n_mb, const int32_t* mb_doc_off,
                                       const int64_t* doc_len, const int64_t* mb_tok_off,
                                       int32_t cp, int32_t policy, const double* model,
                                       int32_t max_segs, int32_t max_docs, int32_t* choice,
                                       double* rank_latency, int64_t* rank_pairs,
                                       int32_t* seg_count, int32_t* segs, int32_t* rowset_off,
                                       int32_t* gather_index, int32_t* positions,
                                       int64_t* features, void* stream) {
  WLB_REQUIRE(cp >= 1 && cp <= kMaxModelCp, "cp must be in [1, %d] for the measured policy",
              kMaxModelCp);
  WLB_REQUIRE(policy == WLB_STRATEGY_PER_SEQUENCE || policy == WLB_STRATEGY_PER_DOCUMENT ||
                  policy == WLB_POLICY_MEASURED,
              "unknown policy %d", policy);
  WLB_REQUIRE(model != nullptr, "model is required");
  return launch_plan(n_mb, mb_doc_off, doc_len, mb_tok_off, cp, policy, 1, nullptr, nullptr, 0,
                     1.0, max_segs, max_docs, choice, rank_latency, rank_pairs, seg_count, segs,
                     rowset_off, gather_index, positions, model, features, (cudaStream_t)stream);
}

extern "C" int wlb_kernel_latency_sum(const int64_t* q_lens, const int64_t* kv_lens, int64_t n,
                                      int64_t tile, const int64_t* curve_q, const double* curve_v,
                                      int32_t n_curve, double op_scale, double* out, void* stream) {
  WLB_REQUIRE(n >= 0 && n_curve >= 1 && tile >= 1, "bad arguments");
  kernel_latency_sum_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      (const long long*)q_lens, (const long long*)kv_lens, n, tile, (const long long*)curve_q,
      curve_v, n_curve, op_scale, out);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

// Scratch for the unsorted items lives right after the sorted array.
extern "C" int wlb_attn_tiles(int32_t n_docs, const int32_t* rowset_off, const int32_t* positions,
                              const int32_t* doc_start, int32_t block_m, int32_t max_tiles,
                              int32_t* tiles, int32_t* n_tiles, void* stream) {
  WLB_REQUIRE(block_m == 128, "block_m must be 128");
  WLB_REQUIRE(n_docs >= 0 && max_tiles >= 1, "bad arguments");
  attn_tiles_kernel<<<1, kTileThreads, 0, (cudaStream_t)stream>>>(
      n_docs, rowset_off, positions, doc_start, block_m, max_tiles, (int4*)tiles, n_tiles,
      (int4*)tiles + 2 * (size_t)max_tiles);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}
