// Bucket-centric join (the default E_loc path for single-sector sample sets).
//
// The deletion index (qvmc_join.cuh) groups the entries (y, T_y) into exact
// buckets; a bucket with k members holds k rows that all need all k members
// as candidates, so the search work is sum_B k_B^2 (94% of it in buckets with
// k >= 33 at 118 qubits, 1e6 samples). The row-centric walk pays a cursor
// advance, a member load and a decode per candidate; here a warp owns a
// (bucket, row range) work item, the rows are warp-uniform and the lanes run
// over the bucket's members (L1-resident for the whole item), so a candidate
// costs one L1 load, the accept rule and one existence-bitmap test.
//
// Output, per member entry p = (row i, bucket B): the hits of row i in B as a
// chain of chunks (normally one). Evaluation runs per row afterwards
// (k_bucket_eval): its chunks in pair order t = 0..C-1, so E_loc sums in a
// fixed order (deterministic), with the row's diagonal and residual parts.
#pragma once

#include "qvmc_join.cuh"

namespace qvmc_b200 {

#ifndef QVMC_BUCKET_MINB
#define QVMC_BUCKET_MINB 5
#endif
#ifndef QVMC_BUCKET_UNROLL
#define QVMC_BUCKET_UNROLL 2  // members per lane in flight
#endif
#ifndef QVMC_BEVAL_MINB
#define QVMC_BEVAL_MINB 4
#endif
constexpr uint32_t kItemWork = 1u << 14;  // target candidate pairs per work item
constexpr int kBQueue = 256;              // per-warp hit queue of the search
constexpr int kBFlushAt = kBQueue - 32 * (QVMC_BUCKET_UNROLL + 1);  // the survivors of one step + a lookup batch
constexpr int kBList = 512;               // per-warp chunk list of the evaluation (segmented beyond)

// rows per work item of a bucket with k members
__host__ __device__ __forceinline__ uint32_t item_rows(uint32_t k) {
  const uint32_t r = (kItemWork + k - 1) / k;
  return r < 1 ? 1 : r;
}

// work items per run (bucket): buckets of one member have no candidates
__global__ void k_item_count(const uint32_t* __restrict__ run_lo, const uint32_t* __restrict__ run_hi,
                             const uint32_t* __restrict__ rid, uint64_t E, uint32_t* __restrict__ cnt) {
  const uint32_t n_runs = E ? rid[E - 1] : 0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < E; r += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (r < n_runs) {
      const uint32_t k = run_hi[r] - run_lo[r];
      if (k >= 2) c = (k + item_rows(k) - 1) / item_rows(k);
    }
    cnt[r] = c;
  }
}

// item = (bucket lo, bucket hi, first row position, end row position)
__global__ void k_item_emit(const uint32_t* __restrict__ run_lo, const uint32_t* __restrict__ run_hi,
                            const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ incl, uint64_t E,
                            uint4* __restrict__ items) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < E; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cnt[r];
    if (!c) continue;
    const uint32_t lo = run_lo[r], hi = run_hi[r], R = item_rows(hi - lo);
    const uint32_t base = incl[r] - c;
    for (uint32_t q = 0; q < c; ++q) items[base + q] = make_uint4(lo, hi, lo + q * R, min(hi, lo + (q + 1) * R));
  }
}

struct BucketOut {
  uint32_t* hy;  // [hit_cap] partner (key-array position)
  uint32_t* hg;  // [hit_cap] group
  uint32_t* hk;  // [hit_cap] flip position key
  uint4* chunk;  // [chunk_cap] (first hit, hits, next chunk of the same entry or ~0, 0)
  uint32_t* head;  // [E] first chunk of the entry or ~0 (memset 0xFF)
  unsigned long long* hit_cursor;
  unsigned long long* chunk_cursor;
  uint64_t hit_cap, chunk_cap;
};

constexpr int kSurv = 128;  // per-warp ring of bitmap survivors awaiting their flip-table lookup

struct BucketSmem {
  uint32_t qy[kBQueue];  // hit queue of the current row: partner, group, flip position key
  uint32_t qg[kBQueue];
  uint32_t qk[kBQueue];
  uint32_t sy[kSurv];    // survivors (partner, flip position key), looked up 32 at a time
  uint32_t sk[kSurv];
  unsigned qn;
};

// Output space is reserved per warp in blocks (one global atomic per block,
// not per chunk: a chunk per (row, bucket) would put tens of millions of
// atomics on two addresses); the unused tail of a block is left as a gap.
constexpr uint64_t kHitBlock = 4096;
constexpr uint64_t kChunkBlock = 256;

struct WarpAlloc {
  uint64_t hit_next = 0, hit_end = 0;
  uint64_t chunk_next = 0, chunk_end = 0;
};

// flush the queue as one chunk of entry p (chained after `prev`, or head[p])
__device__ __forceinline__ void bucket_flush(BucketSmem* sm, const BucketOut& O, const Ctl& C, uint32_t p,
                                             uint32_t& prev, WarpAlloc& A, int lane) {
  __syncwarp();
  const unsigned qn = sm->qn;
  if (A.hit_next + qn > A.hit_end) {  // warp-uniform
    const uint64_t want = qn > kHitBlock ? qn : kHitBlock;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(O.hit_cursor, static_cast<unsigned long long>(want));
    A.hit_next = __shfl_sync(0xffffffffu, b, 0);
    A.hit_end = A.hit_next + want;
  }
  if (A.chunk_next == A.chunk_end) {
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(O.chunk_cursor, static_cast<unsigned long long>(kChunkBlock));
    A.chunk_next = __shfl_sync(0xffffffffu, b, 0);
    A.chunk_end = A.chunk_next + kChunkBlock;
  }
  const uint64_t off = A.hit_next, cid = A.chunk_next;
  A.hit_next += qn;
  A.chunk_next += 1;
  if (off + qn <= O.hit_cap && cid < O.chunk_cap) {
    for (unsigned k = lane; k < qn; k += 32) {
      O.hy[off + k] = sm->qy[k];
      O.hg[off + k] = sm->qg[k];
      O.hk[off + k] = sm->qk[k];
    }
    if (lane == 0) {
      O.chunk[cid] = make_uint4(static_cast<uint32_t>(off), qn, ~0u, 0u);
      if (prev == ~0u) O.head[p] = static_cast<uint32_t>(cid);
      else O.chunk[prev].z = static_cast<uint32_t>(cid);
    }
    prev = static_cast<uint32_t>(cid);
  } else if (lane == 0) {
    atomicOr(C.err, kErrHitOverflow);  // the host grows the buffers and reruns
  }
  __syncwarp();
  if (lane == 0) sm->qn = 0;
  __syncwarp();
}

// look up the flip masks of up to 32 survivors (one per lane, dense) and
// append the hits to the row's queue
__device__ __forceinline__ void lookup_survivors(BucketSmem* sm, const JoinView& J, uint32_t head, uint32_t count,
                                                 int lane, uint32_t& hits) {
  const bool valid = static_cast<uint32_t>(lane) < count;
  uint32_t y = 0, key = kNoKey;
  int64_t g = -1;
  if (valid) {
    const uint32_t e = (head + lane) & (kSurv - 1);
    y = sm->sy[e];
    key = sm->sk[e];
    const uint32_t bk = xy_bucket(key, static_cast<uint32_t>(J.xy_mask));
    g = xy_resolve(key, ldg256(J.xy_tab + static_cast<uint64_t>(bk) * 4));
    if (g == kChain) g = xy_chain(key, bk, J.xy_tab, static_cast<uint32_t>(J.xy_mask));
  }
  const bool hit = g >= 0;
  const unsigned hm = __ballot_sync(0xffffffffu, hit);
  if (hm) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&sm->qn, __popc(hm));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (hit) {
      const unsigned k = base + __popc(hm & ((1u << lane) - 1u));
      sm->qy[k] = y;
      sm->qg[k] = static_cast<uint32_t>(g);
      sm->qk[k] = key;
    }
    hits += __popc(hm);
  }
  __syncwarp();
}

template <int W>
__global__ void __launch_bounds__(kThreads, QVMC_BUCKET_MINB)
    k_bucket_search(const __grid_constant__ JoinView J, const uint64_t* __restrict__ keys, int n_qubits,
                    const uint4* __restrict__ items, const uint32_t* __restrict__ n_items_p, int side,
                    const uint32_t* __restrict__ perm, int64_t r_begin, int64_t r_end,
                    const __grid_constant__ Ctl C, const __grid_constant__ BucketOut O) {
  __shared__ BucketSmem s_w[kWarps];
  const int lane = threadIdx.x & 31;
  BucketSmem* sm = &s_w[threadIdx.x >> 5];
  if (lane == 0) sm->qn = 0;
  __syncwarp();
  const uint32_t n_items = *n_items_p;
  uint64_t tot_cand = 0, tot_hits = 0;
  WarpAlloc A;
  for (;;) {
    unsigned long long it_id = 0;
    if (lane == 0) it_id = atomicAdd(C.row_next, 1ull);
    it_id = __shfl_sync(0xffffffffu, it_id, 0);
    if (it_id >= n_items) break;
    const uint4 it = __ldg(items + it_id);
    const uint32_t lo = it.x, hi = it.y;
    // the bucket's common set R = S(y) - T_y of any member: its two smallest
    // orbitals decide the single-excitation accept rule of every row
    int r0 = 0x7FFF, r1 = 0x7FFF;
    {
      const uint64_t v0 = __ldg(J.mem + lo);
      const int64_t y0 = static_cast<uint32_t>(v0);
      const int a0 = static_cast<int>(v0 >> 32) & 0xFF, b0 = static_cast<int>(v0 >> 40) & 0xFF;
      int got = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t v = side ? __ldg(keys + y0 * W + w) : ~__ldg(keys + y0 * W + w);
        const int hi_bit = n_qubits - 64 * w;
        if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
        while (v && got < 2) {
          const int q = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
          v &= v - 1;
          if (q == a0 || q == b0) continue;
          if (got == 0) r0 = q;
          else r1 = q;
          ++got;
        }
      }
    }
    for (uint32_t p = it.z; p < it.w; ++p) {  // the item's rows (warp-uniform)
      const uint64_t vi = __ldg(J.mem + p);
      if (perm) {  // a row shard: rows of other ranks are skipped
        const int64_t orow = __ldg(perm + static_cast<uint32_t>(vi));
        if (orow < r_begin || orow >= r_end) continue;
      }
      const int ta = static_cast<int>(vi >> 32) & 0xFF, tb = static_cast<int>(vi >> 40) & 0xFF;
      const uint32_t dbase = J.P + static_cast<uint32_t>(vi >> 48) * J.P;
      // two smallest orbitals of S(x) = R + {ta, tb} (ta < tb)
      int pos0, pos1;
      if (ta < r0) {
        pos0 = ta;
        pos1 = tb < r0 ? tb : r0;
      } else {
        pos0 = r0;
        pos1 = ta < r1 ? ta : r1;
      }
      uint32_t prev = ~0u;
      uint32_t hits = 0;
      uint32_t s_head = 0, s_tail = 0;  // survivor ring (warp-uniform)
      for (uint32_t j0 = lo; j0 < hi; j0 += 32 * QVMC_BUCKET_UNROLL) {
        constexpr int U = QVMC_BUCKET_UNROLL;
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + 32 * u + lane;
          v[u] = j < hi ? __ldg(J.mem + j) : ~0ull;
        }
        // accept rule + existence bitmap; survivors go to the ring (dense lookups later)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t key = kNoKey;
          if (v[u] != ~0ull) {
            const int ya = static_cast<int>(v[u] >> 32) & 0xFF, yb = static_cast<int>(v[u] >> 40) & 0xFF;
            const bool ea = ya == ta || ya == tb, eb = yb == ta || yb == tb;
            if (!ea && !eb) {  // double excitation
              ++tot_cand;
              if (!J.pbits || pbit(J.pbits, dbase + static_cast<uint32_t>(v[u] >> 48))) {
                int p0 = ta, p1 = tb, p2 = ya, p3 = yb;
                sort2(p0, p2);
                sort2(p1, p3);
                sort2(p1, p2);
                key = static_cast<uint32_t>(p0) | static_cast<uint32_t>(p1) << 8 | static_cast<uint32_t>(p2) << 16 |
                      static_cast<uint32_t>(p3) << 24;
              }
            } else if (ea != eb) {  // single excitation: x loses cc, gains a; accept once
              const int o = ea ? ya : yb, a = ea ? yb : ya;
              const int cc = (o == ta) ? tb : ta;
              if (o == (cc == pos0 ? pos1 : pos0)) {
                ++tot_cand;
                int p0 = cc, p1 = a;
                sort2(p0, p1);
                if (!J.pbits || pbit(J.pbits, pidx(p0, p1)))
                  key = static_cast<uint32_t>(p0) | static_cast<uint32_t>(p1) << 8 | 0xFFFF0000u;
              }
            }
          }
          const unsigned sm_mask = __ballot_sync(0xffffffffu, key != kNoKey);
          if (key != kNoKey) {
            const uint32_t e = (s_tail + __popc(sm_mask & ((1u << lane) - 1u))) & (kSurv - 1);
            sm->sy[e] = static_cast<uint32_t>(v[u]);
            sm->sk[e] = key;
          }
          s_tail += __popc(sm_mask);
        }
        __syncwarp();
        while (s_tail - s_head >= 32) {
          lookup_survivors(sm, J, s_head, 32, lane, hits);
          s_head += 32;
        }
        if (sm->qn >= static_cast<unsigned>(kBFlushAt)) bucket_flush(sm, O, C, p, prev, A, lane);
      }
      if (s_tail != s_head) lookup_survivors(sm, J, s_head, s_tail - s_head, lane, hits);
      if (sm->qn > 0) bucket_flush(sm, O, C, p, prev, A, lane);
      tot_hits += hits;  // warp total (identical on every lane)
    }
  }
  tot_cand = warp_sum(tot_cand);
  if (lane == 0) {
    atomicAdd(C.stats, static_cast<unsigned long long>(tot_cand));
    atomicAdd(C.stats + 1, static_cast<unsigned long long>(tot_hits));
  }
}

struct BEvalSmem {
  uint32_t l_off[kBList];  // the row's chunks in pair order: first hit, hits
  uint32_t l_len[kBList];
  uint16_t pos[32];
  uint8_t ta[kJoinMaxRanges];
  uint8_t tb[kJoinMaxRanges];
};

// Per-row evaluation of the bucket search's hits (one warp per row):
// diagonal (+ residual masks) + every hit, hits walked in pair order t and
// chunk order; rows whose chunk list exceeds kBList are processed in segments.
template <int W>
__global__ void __launch_bounds__(kThreads, QVMC_BEVAL_MINB)
    k_bucket_eval(const __grid_constant__ HamView H, const TableView T, const __grid_constant__ JoinView J,
                  const uint64_t* __restrict__ keys, const RowSet R, int side, int s, const uint32_t* __restrict__ pos_of,
                  const uint32_t* __restrict__ head, const uint4* __restrict__ chunk, const uint32_t* __restrict__ hy,
                  const uint32_t* __restrict__ hg, const uint32_t* __restrict__ hk, const __grid_constant__ Ctl C,
                  double2* __restrict__ eloc) {
  __shared__ BEvalSmem s_w[kWarps];
  const int lane = threadIdx.x & 31;
  BEvalSmem* sm = &s_w[threadIdx.x >> 5];
  const int n = H.n;
  const int n_ranges = s * (s - 1) / 2;
  for (;;) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(C.row_next, 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (static_cast<int64_t>(r) >= R.n_rows) break;
    const int64_t row = R.list ? static_cast<int64_t>(__ldg(R.list + r)) : R.base + static_cast<int64_t>(r);
    const int64_t orow = R.perm ? static_cast<int64_t>(__ldg(R.perm + row)) : row;

    Key<W> xrow;
#pragma unroll
    for (int w = 0; w < W; ++w) xrow.w[w] = __ldg(keys + row * W + w);
    const U64x4 sr = ldg256(J.rec + row * 4);
    const double la_i = __longlong_as_double(static_cast<long long>(sr.a));
    const double2 cs_i = make_double2(__longlong_as_double(static_cast<long long>(sr.b)),
                                      __longlong_as_double(static_cast<long long>(sr.c)));
    if (isinf(la_i)) {  // energy.cpp:32-33
      if (lane == 0) {
        atomicOr(C.err, kErrZeroAmp);
        eloc[orow - R.out_base] = make_double2(CUDART_NAN, CUDART_NAN);
      }
      continue;
    }
    int pos = 0, cnt = 0;  // lane a < s holds the a-th minority orbital
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint64_t v = side ? xrow.w[w] : ~xrow.w[w];
      const int hi_bit = n - 64 * w;
      if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      const int pc = __popcll(v);
      if (lane >= cnt && lane < cnt + pc) {
        for (int k = 0; k < lane - cnt; ++k) v &= v - 1;
        pos = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
      }
      cnt += pc;
    }
    __syncwarp();
    if (lane < s) sm->pos[lane] = static_cast<uint16_t>(pos);
    __syncwarp();
    for (int t = lane; t < n_ranges; t += 32) {
      const uint32_t b = pair_b(t);
      sm->ta[t] = static_cast<uint8_t>(sm->pos[t - b * (b - 1) / 2]);
      sm->tb[t] = static_cast<uint8_t>(sm->pos[b]);
    }
    __syncwarp();

    double2 acc = make_double2(0.0, 0.0);
    // the row's chunks in (t, chain) order, kBList at a time
    uint32_t total = 0;
    for (uint32_t seg = 0;; seg += kBList) {
      uint32_t base = 0;  // chunks of the t's before this lane's current t
      for (int t0 = 0; t0 < n_ranges; t0 += 32) {
        const int t = t0 + lane;
        uint32_t c = ~0u, len = 0;
        if (t < n_ranges) {
          c = __ldg(head + __ldg(pos_of + static_cast<uint64_t>(row) * J.C + t));
          for (uint32_t q = c; q != ~0u; q = __ldg(chunk + q).z) ++len;
        }
        uint32_t incl = len;  // warp inclusive scan of the chain lengths
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        uint32_t at = base + incl - len;
        for (uint32_t q = c; q != ~0u; ++at) {
          const uint4 ch = __ldg(chunk + q);
          if (at >= seg && at < seg + kBList) {
            sm->l_off[at - seg] = ch.x;
            sm->l_len[at - seg] = ch.y;
          }
          q = ch.z;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
      total = base;
      __syncwarp();
      const int n_list = static_cast<int>(min(total - min(total, seg), static_cast<uint32_t>(kBList)));
      // flattened walk over the listed chunks: lane l takes hits l, l+32, ...
      int rg = 0;
      uint32_t off = lane;
      uint32_t len = n_list > 0 ? sm->l_len[0] : 0;
      while (rg < n_list && off >= len) {
        off -= len;
        if (++rg < n_list) len = sm->l_len[rg];
      }
      while (__any_sync(0xffffffffu, rg < n_list)) {
        JoinHit h;
        h.valid = rg < n_list;
        h.key = kNoKey;
        h.sr = U64x4{0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < kGrecWords; ++i) h.r[i] = 0;
        if (h.valid) {
          const uint64_t at = static_cast<uint64_t>(sm->l_off[rg]) + off;
          const uint32_t y = __ldg(hy + at), g = __ldg(hg + at);
          h.key = __ldg(hk + at);
          h.sr = ldg256(J.rec + static_cast<int64_t>(y) * 4);
          const U64x4 g0 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords);
          const U64x4 g1 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords + 4);
          h.r[0] = g0.a; h.r[1] = g0.b; h.r[2] = g0.c; h.r[3] = g0.d;
          h.r[4] = g1.a; h.r[5] = g1.b; h.r[6] = g1.c; h.r[7] = g1.d;
          off += 32;
          while (rg < n_list && off >= len) {
            off -= len;
            if (++rg < n_list) len = sm->l_len[rg];
          }
        }
        eval_hit<W>(H, J, sm->pos, h, xrow, la_i, cs_i, lane, s, side, acc);
      }
      __syncwarp();
      if (seg + kBList >= total) break;
    }

    // even flip masks of weight >= 6: popcount filter + sample-set probe
    if (H.n_res) {
      uint64_t S[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        S[w] = side ? xrow.w[w] : ~xrow.w[w];
        const int hi_bit = n - 64 * w;
        if (hi_bit < 64) S[w] &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
      }
      const uint64_t hx_res = key_hash_warp<W>(xrow.w, H.hash_bytes, lane);
      for (uint32_t b0 = 0; b0 < H.n_res; b0 += 32) {
        const uint32_t e = b0 + lane;
        if (e < H.n_res) {
          const uint32_t g = __ldg(H.res_g + e);
          int in_s = 0, wt = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint64_t mm = __ldg(H.xy + (int64_t)g * W + w);
            in_s += __popcll(mm & S[w]);
            wt += __popcll(mm);
          }
          if (2 * in_s == wt) {
            const int64_t j = probe_slow<W>(xrow, fmix(hx_res ^ __ldg(H.xy_hash + g)), g, T.tab, T.mask, keys, H.xy);
            if (j >= 0) {
              uint64_t xp[W];
#pragma unroll
              for (int w = 0; w < W; ++w) xp[w] = __ldg(keys + j * W + w);
              double hr, hi;
              group_element<W>(H, xp, g, hr, hi);
              const U64x4 srj = ldg256(J.rec + j * 4);
              add_ratio(__longlong_as_double(static_cast<long long>(srj.a)),
                        make_double2(__longlong_as_double(static_cast<long long>(srj.b)),
                                     __longlong_as_double(static_cast<long long>(srj.c))),
                        la_i, cs_i, hr, hi, acc);
            }
          }
        }
      }
    }

    // diagonal element as the quadratic form over S(x)
    if (H.diag >= 0) {
      if (H.diag_quad) {
        if (lane == 0) acc.x += side ? H.diag_A1 : H.diag_A0;
        if (lane < s) acc.x += __ldg(H.diag_b + side * n + pos);
        for (int pi = lane; pi < n_ranges; pi += 32) acc.x += __ldg(H.diag_K + sm->ta[pi] * n + sm->tb[pi]);
        for (uint32_t e = lane; e < H.n_diag_other; e += 32) {
          const uint32_t t = __ldg(H.diag_other + e);
          int pc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) pc += __popcll(xrow.w[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int qt = (__ldg(H.yw + t) + 2 * pc) & 3;
          const double cf = __ldg(H.coeff + t);
          if (qt == 0) acc.x += cf;
          else if (qt == 2) acc.x -= cf;
          else if (qt == 1) acc.y += cf;
          else acc.y -= cf;
        }
      } else {
        const uint32_t t1 = __ldg(H.goff + H.diag + 1);
        for (uint32_t t = __ldg(H.goff + H.diag) + lane; t < t1; t += 32) {
          int pc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) pc += __popcll(xrow.w[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int qt = (__ldg(H.yw + t) + 2 * pc) & 3;
          const double cf = __ldg(H.coeff + t);
          if (qt == 0) acc.x += cf;
          else if (qt == 2) acc.x -= cf;
          else if (qt == 1) acc.y += cf;
          else acc.y -= cf;
        }
      }
    }
    const double re = warp_sum(acc.x);
    const double im = warp_sum(acc.y);
    if (lane == 0) {
      eloc[orow - R.out_base] = make_double2(re, im);
      if (H.diag >= 0) atomicAdd(C.stats + 1, 1ull);  // the diagonal pair, counted like the row kernels
    }
  }
}

}  // namespace qvmc_b200
