// libqvmc_cuda: C ABI (include/qvmc_cuda.h) over the sm_100a kernels in
// qvmc_kernels.cuh. Host code here only validates, sizes workspaces, copies
// and launches; there is no CPU compute path for the per-sample work.
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <cub/device/device_segmented_sort.cuh>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_index.h"
#include "qvmc_comm.cuh"
#include "qvmc_cuda.h"
#include "qvmc_join.cuh"
#include "qvmc_kernels.cuh"
#include "qvmc_model.cuh"
#include "qvmc_sampler.cuh"

using namespace qvmc_b200;

namespace {

thread_local std::string g_error;
std::atomic<uint64_t> g_launches{0};

struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(QVMC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void ck_launch(const char* what) {
  ++g_launches;
  ck(cudaGetLastError(), what);
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return QVMC_OK;
  } catch (const Failure& e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return QVMC_ERR_INVALID_ARGUMENT;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return QVMC_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_error = e.what();
    return QVMC_ERR_RUNTIME;
  }
}

// restores the caller's current device on scope exit
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    ck(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// grow-only device buffer
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t want) {
    if (want <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    ck(cudaMalloc(&p, want), "cudaMalloc");
    bytes = want;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

template <typename T>
void upload(DBuf& b, const std::vector<T>& v) {
  b.ensure(std::max<size_t>(v.size() * sizeof(T), 16));
  if (!v.empty()) ck(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
}

}  // namespace

struct qvmc_index_s {
  HostIndex idx;
};

struct qvmc_comm_s {
  int world = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  bool owns = false;                      // created here (destroyed with the comm)
  qvmc_host_allgather_fn host_ag = nullptr;  // host backend
  void* ctx = nullptr;
  void* hsend = nullptr;                  // pinned staging of the host backend
  void* hrecv = nullptr;
  size_t hsend_bytes = 0, hrecv_bytes = 0;
};

namespace {

void nccl_ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(QVMC_ERR_RUNTIME, std::string(what) + ": " + nccl_api().GetErrorString(r));
}

const NcclApi& nccl_or_fail() {
  const NcclApi& a = nccl_api();
  if (a.error) fail(QVMC_ERR_RUNTIME, a.error);
  return a;
}

void pinned_ensure(void*& p, size_t& have, size_t want) {
  if (want <= have) return;
  if (p) cudaFreeHost(p);
  p = nullptr;
  have = 0;
  ck(cudaMallocHost(&p, want), "cudaMallocHost");
  have = want;
}

// all-gather `bytes` per rank (multiple of 8) from device send to device recv on `stream`
void comm_all_gather(qvmc_comm_s* c, const void* send, void* recv, size_t bytes, cudaStream_t stream) {
  if (c->nccl) {
    nccl_ck(nccl_api().AllGather(send, recv, bytes / 8, ncclUint64, c->nccl, stream), "ncclAllGather");
    return;
  }
  pinned_ensure(c->hsend, c->hsend_bytes, std::max<size_t>(bytes, 8));
  pinned_ensure(c->hrecv, c->hrecv_bytes, std::max<size_t>(bytes * c->world, 8));
  if (bytes) ck(cudaMemcpyAsync(c->hsend, send, bytes, cudaMemcpyDeviceToHost, stream), "D2H shard");
  ck(cudaStreamSynchronize(stream), "sync");
  if (c->host_ag(c->ctx, c->hsend, c->hrecv, bytes) != 0) fail(QVMC_ERR_RUNTIME, "host all-gather callback failed");
  if (bytes) ck(cudaMemcpyAsync(recv, c->hrecv, bytes * c->world, cudaMemcpyHostToDevice, stream), "H2D gathered");
}

// in-place sum over the ranks of a uint64 array (exact: integer); the host backend all-gathers into tmp
void comm_all_reduce_u64(qvmc_comm_s* c, unsigned long long* buf, size_t count, cudaStream_t stream, DBuf& tmp) {
  if (c->world == 1 || count == 0) return;
  if (c->nccl) {
    nccl_ck(nccl_api().AllReduce(buf, buf, count, ncclUint64, ncclSum, c->nccl, stream), "ncclAllReduce");
    return;
  }
  tmp.ensure(count * 8 * c->world + 16);
  comm_all_gather(c, buf, tmp.p, count * 8, stream);
  k_sum_ranks_u64<<<static_cast<int>(std::min<size_t>((count + 255) / 256, 4096)), 256, 0, stream>>>(
      tmp.as<unsigned long long>(), c->world, static_cast<int64_t>(count), buf);
  ck_launch("sum ranks");
}

}  // namespace

struct qvmc_ham_s {
  int device = 0;
  int n = 0, W = 0;
  uint32_t n_xy = 0;
  int64_t diag = -1;
  uint64_t n_terms = 0;
  int sms = 148;
  cudaStream_t own = nullptr, stream = nullptr;
  // Hamiltonian
  DBuf xy, xy_hash, goff, coeff, yz, yw, xyw, gen_hash, gen_g, lst_off, lst_hash, lst_g, res_g, diag_b, diag_K,
      diag_other, hash_bytes, xy_tab, codes, comp_of, fam_off, fam_B, fam_q, fam_u, fam_V, fam_v, ginfo, trec,
      famrec, grec, famvi, pbits, binom;
  std::vector<uint64_t> binom_host;
  uint64_t xy_tab_mask = 0;
  uint32_t pbits_P = 0;
  DBuf hot;  // grec | famvi | pbits | xy_tab in one arena
  size_t hot_bytes = 0;
  uint64_t* p_grec = nullptr;
  double* p_famvi = nullptr;
  uint32_t* p_pbits = nullptr;
  uint64_t* p_xy_tab = nullptr;
  HamView view{};
  // join path (per call): deletion-index workspace
  DBuf l_key, l_key2, l_idx, l_perm, l_keys, l_rec, l_flags, l_list, l_nsel, cs;
  DBuf j_key, j_val, j_key2, j_val2, j_head, j_rid, j_lo, j_hi, j_mem, j_rng, j_tmp;
  bool use_join = true;
  // split-evaluation workspace
  DBuf s_row_last, s_base, s_rowpos;
  uint64_t hits_per_row = 320;  // split evaluation: running estimate that sizes the row batches
  // speculative device-memory calls (no host synchronisation): the last call's sector plan,
  // checked on the device; a call that needs a re-plan or larger hit buffers is rerun by the
  // next qvmc_cuda_synchronize with the arguments kept here
  bool plan_ok = false;
  int plan_mm[2] = {0, 0};
  int64_t plan_n = -1;
  bool plan_sector = false, plan_join = false;
  int plan_side = 0, plan_s = 0, plan_key_bits = 0;
  bool no_spec = true;  // speculation is opt-in: qvmc_cuda_set_speculative / QVMC_SPECULATE=1
  bool pending = false;
  struct {
    int64_t n_unq, r0, r1;
    const uint64_t* keys;
    const double *la, *ph, *lp;
    double log_norm;
    double *eloc, *moments;
  } pend{};
  int64_t pend_nb = 0;
  cudaStream_t pend_stream = nullptr;  // the stream the speculative call ran on
  DBuf gkey, p_rlo, p_rhi;      // per-group position key (pairs-based local_energies), row ranges
  // pipelined split evaluation (run_join_pipelined)
  DBuf p_hy[2], p_hg[2], p_hk[2], p_chunk[2], p_part[2];
  uint64_t p_hit_cap = 0, p_chunk_cap = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_p[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  unsigned long long* log_host = nullptr;
  uint64_t log_cap = 0;
  int pipe_batches = 2, pipe_search_blocks = 0, pipe_eval_blocks = 0;  // measured: 2-3 batches best
  // workspace
  DBuf tab, ctl, keys, la, ph, lp, eloc, partials, moments, weights;
  DBuf counts, row_off, xp_a, g_a, xp_b, g_b, entries, cub_tmp, in_entries, out_h, out_class;
  DBuf s_keys, s_la, s_ph, s_lp, g_send, g_recv, g_keys, g_la, g_ph, g_lp, g_mom, g_moms;  // sharded calls
  uint64_t tab_buckets = 0;
  uint64_t n_pairs = 0;
  int64_t pairs_rows = 0;
  qvmc_stats last{};
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // fused-call stage timing
  bool timed = false;
  std::vector<cudaEvent_t> ev_b;  // pipelined split evaluation: per batch search start/end, eval start/end
  cudaEvent_t ev_f[2] = {nullptr, nullptr};  // fused join kernel start/end
  bool timed_f = false;
  bool sym = true;     // QVMC_SYMMETRIC=0: every row walks all its partners (no exchange symmetry)
  bool sym_last = false;  // the last index build was symmetric
  DBuf s_fix;             // symmetric mode: per row 2 x 128-bit fixed-point sums of mirrored contributions
  bool shard_sym_active = false;  // the last fused call left its mirrored sums in s_fix
  qvmc_comm_s* dist_comm = nullptr;  // set by qvmc_cuda_eloc_sharded: build the deletion index across ranks
  bool dist_index = true;            // QVMC_DIST_INDEX=0: every rank builds the whole index
  bool dist_active = false;          // the last index was built across ranks (members in j_memg)
  DBuf j_flags, j_count, j_memg, j_rtmp;
  bool sym_off_once = false;  // the next call evaluates unpaired (a fixed-point range fallback)
  bool fix_range_flag = false;  // a sharded symmetric call left the fixed-point range
  bool shard_sym = false;  // set by qvmc_cuda_eloc_sharded: symmetric over a row subset, mirrored sums
                           // left in s_fix for the cross-rank reduction (not added by finalize)
  RowSet last_rows{};      // the row set of the last fused call (sorted positions -> caller rows)
  bool fused = false;  // QVMC_FUSED=1: one warp-specialised search + evaluation kernel (measured slower, r2a)
  bool strided_shards = true;  // QVMC_STRIDED_SHARDS=0: a sharded call walks its own (contiguous) caller rows
  int walk_world = 0, walk_rank = 0;  // set by qvmc_cuda_eloc_sharded: walk sorted positions rank, rank + world, ...
  int64_t timed_b = 0;            // batches timed by ev_b in the last call
};

// the speculative-call rerun (resolve_pending) calls the C entry point
extern "C" int qvmc_cuda_eloc_fused(qvmc_ham_t, int64_t, const uint64_t*, const double*, const double*,
                                    const double*, double, int64_t, int64_t, double*, double*, int);

namespace {

constexpr int kCtlInts = 16;  // int err, pad, popc_mm[2]; u64 row_next @4, stats[2] @6, hit/chunk cursors @10/@12,
                              // int exp flag @14 (some |log psi| > 700)

Ctl ctl_view(qvmc_ham_s* h) {
  Ctl c;
  int* base = h->ctl.as<int>();
  c.err = base;
  c.popc_mm = base + 2;
  c.row_next = reinterpret_cast<unsigned long long*>(base + 4);
  c.stats = reinterpret_cast<unsigned long long*>(base + 6);
  return c;
}

void check_handle(qvmc_ham_s* h) {
  if (!h) fail(QVMC_ERR_INVALID_ARGUMENT, "null qvmc handle");
}

int grid_for(qvmc_ham_s* h, int per_sm) { return std::max(1, h->sms * std::max(1, per_sm)); }

// ------------------------------------------------------------- small kernels

__global__ void k_fill_u64(uint64_t* p, uint64_t n, uint64_t v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// row ranges of a canonical pair list (sorted by x): row_lo / row_hi (memset 0 first)
__global__ void k_pair_rows(const uint32_t* __restrict__ e3, uint64_t n_pairs, int64_t n, uint32_t* row_lo,
                            uint32_t* row_hi) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_pairs;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = e3[3 * e];
    if (x >= n) continue;  // reported by k_check_sorted
    if (e == 0 || e3[3 * (e - 1)] != x) row_lo[x] = static_cast<uint32_t>(e);
    if (e + 1 == n_pairs || e3[3 * (e + 1)] != x) row_hi[x] = static_cast<uint32_t>(e + 1);
  }
}

// local_energies from a canonical pair list (energy.cpp:13-48), one warp per
// row: H_{x x'} from the 64-byte drain records when x' = x ^ xy (kind A
// bit-identical to group_element; kind B for single moves within the row's
// minority set), term by term otherwise (the reference evaluates whatever x'
// an entry names); phases from per-sample (cos, sin).
template <int W>
__global__ void __launch_bounds__(kThreads)
    k_pairs_eloc2(const __grid_constant__ HamView H, const __grid_constant__ JoinView J, const uint32_t* __restrict__ gkey,
                  const uint64_t* __restrict__ keys, const double* __restrict__ la, const double2* __restrict__ cs,
                  int64_t n, const uint32_t* __restrict__ e3, const uint32_t* __restrict__ row_lo,
                  const uint32_t* __restrict__ row_hi, double2* out, int* err) {
  __shared__ uint16_t s_pos[kWarps][32];
  const int lane = threadIdx.x & 31;
  uint16_t* spos = s_pos[threadIdx.x >> 5];
  const int nq = H.n;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += n_warps) {
    const double la_i = la[i];
    if (isinf(la_i)) {
      if (lane == 0) {
        atomicOr(err, kErrZeroAmp);
        out[i] = make_double2(CUDART_NAN, CUDART_NAN);
      }
      continue;
    }
    const double2 cs_i = cs[i];
    Key<W> xrow;
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      xrow.w[w] = keys[i * W + w];
      pc += __popcll(xrow.w[w]);
    }
    const int side = 2 * pc <= nq ? 1 : 0;
    const int s = side ? pc : nq - pc;
    if (s <= 32) {  // the row's minority orbitals (kind B)
      int pos = 0, cnt = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t v = side ? xrow.w[w] : ~xrow.w[w];
        const int hi_bit = nq - 64 * w;
        if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
        const int c = __popcll(v);
        if (lane >= cnt && lane < cnt + c) {
          for (int k = 0; k < lane - cnt; ++k) v &= v - 1;
          pos = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
        }
        cnt += c;
      }
      __syncwarp();
      if (lane < s) spos[lane] = static_cast<uint16_t>(pos);
      __syncwarp();
    }
    const uint32_t lo = row_lo[i], hi = row_hi[i];
    double2 acc = make_double2(0.0, 0.0);
    const bool quad = H.diag >= 0 && H.diag_quad && s <= 32;
    bool has_diag = false;  // the (x, x, diagonal) entry: the warp evaluates it as the quadratic form
    for (uint32_t e0 = lo; e0 < hi; e0 += 32) {
      const uint32_t e = e0 + lane;
      bool valid = e < hi;
      uint32_t j = 0, g = 0;
      if (valid) {
        j = e3[3 * static_cast<uint64_t>(e) + 1];
        g = e3[3 * static_cast<uint64_t>(e) + 2];
        if (j >= n || g >= H.n_xy) {
          atomicOr(err, kErrBadPair);
          valid = false;
        } else if (quad && static_cast<int64_t>(g) == H.diag && static_cast<int64_t>(j) == i) {
          has_diag = true;
          valid = false;
        }
      }
      double hr = 0.0, hi2 = 0.0, la_j = 0.0;
      double2 cs_j = make_double2(1.0, 0.0);
      if (valid) {
        uint64_t xp[W];
#pragma unroll
        for (int w = 0; w < W; ++w) xp[w] = __ldg(keys + static_cast<int64_t>(j) * W + w);
        la_j = __ldg(la + j);
        cs_j = __ldg(cs + j);
        const uint32_t key = __ldg(gkey + g);
        const U64x4 g0 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords);
        const uint32_t kind = static_cast<uint32_t>(g0.a) & 3u;
        bool fast = false;
        if (key != kNoKey && (kind == kGrecA || kind == kGrecB)) {
          uint64_t m[W];
          key_mask<W>(key, m);
          bool is_move = true;  // x' = x ^ xy
#pragma unroll
          for (int w = 0; w < W; ++w) is_move &= xp[w] == (xrow.w[w] ^ m[w]);
          if (kind == kGrecB) {  // a single move inside the minority picture: one flip bit in S(x)
            const bool b0 = bit_at<W>(xrow.w, key & 0xFF) == (side != 0);
            const bool b1 = bit_at<W>(xrow.w, (key >> 8) & 0xFF) == (side != 0);
            is_move &= (b0 != b1) && s <= 32;
          }
          fast = is_move;
        }
        if (fast) {
          const U64x4 g1 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords + 4);
          const uint64_t r[kGrecWords] = {g0.a, g0.b, g0.c, g0.d, g1.a, g1.b, g1.c, g1.d};
          if (kind == kGrecA) kind_a_element<W>(r, xrow.w, key, hr, hi2);
          else kind_b_element<W>(J.famvi, r, xrow.w, key, spos, s, side, hr, hi2);
        } else {
          group_element<W>(H, xp, g, hr, hi2);
        }
        add_ratio(la_j, cs_j, la_i, cs_i, hr, hi2, acc);
      }
    }
    if (__any_sync(0xffffffffu, has_diag)) {  // A + sum_S b_p + sum_{p<q in S} K_pq (+ |z| >= 3 terms)
      if (lane == 0) acc.x += side ? H.diag_A1 : H.diag_A0;
      if (lane < s) acc.x += __ldg(H.diag_b + side * nq + spos[lane]);
      const int np = s * (s - 1) / 2;
      for (int pi = lane; pi < np; pi += 32) {
        const int b = static_cast<int>(pair_b(pi)), a = pi - b * (b - 1) / 2;
        acc.x += __ldg(H.diag_K + spos[a] * nq + spos[b]);
      }
      for (uint32_t e = lane; e < H.n_diag_other; e += 32) {
        const uint32_t t = __ldg(H.diag_other + e);
        int c = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) c += __popcll(xrow.w[w] & __ldg(H.yz + (int64_t)t * W + w));
        const int qt = (__ldg(H.yw + t) + 2 * c) & 3;
        const double cf = __ldg(H.coeff + t);
        if (qt == 0) acc.x += cf;
        else if (qt == 2) acc.x -= cf;
        else if (qt == 1) acc.y += cf;
        else acc.y -= cf;
      }
    }
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    if (lane == 0) out[i] = acc;
  }
}

// Per pair (x, x', xy) of a canonical list: H_{x x'} through the FUSED path's
// evaluators — the 64-byte drain records (kinds A-D, hit_element) when x' =
// x ^ xy is a weight-2/4 flip-table mask, the diagonal as the quadratic form
// over S(x) — plus which evaluator ran (kind: 0-3 = drain record A-D, 4 =
// term by term, 5 = diagonal quadratic form). One warp per row.
template <int W>
__global__ void __launch_bounds__(kThreads)
    k_pair_records(const __grid_constant__ HamView H, const __grid_constant__ JoinView J,
                   const uint32_t* __restrict__ gkey, const uint64_t* __restrict__ keys, int64_t n,
                   const uint32_t* __restrict__ e3, const uint32_t* __restrict__ row_lo,
                   const uint32_t* __restrict__ row_hi, double2* out_h, uint8_t* out_kind, int* err) {
  __shared__ uint16_t s_pos[kWarps][32];
  const int lane = threadIdx.x & 31;
  uint16_t* spos = s_pos[threadIdx.x >> 5];
  const int nq = H.n;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += n_warps) {
    Key<W> xrow;
    int pc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      xrow.w[w] = keys[i * W + w];
      pc += __popcll(xrow.w[w]);
    }
    const int side = 2 * pc <= nq ? 1 : 0;
    const int s = side ? pc : nq - pc;
    int pos = 0;
    if (s <= 32) {
      int cnt = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t v = side ? xrow.w[w] : ~xrow.w[w];
        const int hi_bit = nq - 64 * w;
        if (hi_bit < 64) v &= (hi_bit <= 0) ? 0ull : ((1ull << hi_bit) - 1);
        const int c = __popcll(v);
        if (lane >= cnt && lane < cnt + c) {
          for (int k = 0; k < lane - cnt; ++k) v &= v - 1;
          pos = 64 * w + __ffsll(static_cast<long long>(v)) - 1;
        }
        cnt += c;
      }
      __syncwarp();
      if (lane < s) spos[lane] = static_cast<uint16_t>(pos);
      __syncwarp();
    }
    const bool quad = H.diag >= 0 && H.diag_quad && s <= 32;
    const uint32_t lo = row_lo[i], hi = row_hi[i];
    for (uint32_t e0 = lo; e0 < hi; e0 += 32) {
      const uint32_t e = e0 + lane;
      bool valid = e < hi;
      uint32_t j = 0, g = 0;
      if (valid) {
        j = e3[3 * static_cast<uint64_t>(e) + 1];
        g = e3[3 * static_cast<uint64_t>(e) + 2];
        if (j >= n || g >= H.n_xy) {
          atomicOr(err, kErrBadPair);
          valid = false;
        }
      }
      const bool is_diag = valid && quad && static_cast<int64_t>(g) == H.diag && static_cast<int64_t>(j) == i;
      JoinHit hit;
      hit.valid = false;
      hit.key = kNoKey;
      hit.sr = U64x4{0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < kGrecWords; ++k) hit.r[k] = 0;
      uint8_t kind = 4;
      uint64_t xp[W];
#pragma unroll
      for (int w = 0; w < W; ++w) xp[w] = 0;
      if (valid && !is_diag) {
#pragma unroll
        for (int w = 0; w < W; ++w) xp[w] = __ldg(keys + static_cast<int64_t>(j) * W + w);
        const uint32_t key = __ldg(gkey + g);
        if (key != kNoKey) {
          uint64_t m[W];
          key_mask<W>(key, m);
          bool is_move = true;  // x' = x ^ xy
#pragma unroll
          for (int w = 0; w < W; ++w) is_move &= xp[w] == (xrow.w[w] ^ m[w]);
          const U64x4 g0 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords);
          const U64x4 g1 = ldg256(J.grec + static_cast<int64_t>(g) * kGrecWords + 4);
          const uint32_t kd = static_cast<uint32_t>(g0.a) & 3u;
          if (kd == kGrecB || kd == kGrecD) {  // family forms need a move inside the minority picture
            const bool b0 = bit_at<W>(xrow.w, key & 0xFF) == (side != 0);
            const bool b1 = bit_at<W>(xrow.w, (key >> 8) & 0xFF) == (side != 0);
            is_move &= (kd == kGrecD || b0 != b1) && s <= 32;
          }
          if (is_move) {
            hit.valid = true;
            hit.key = key;
            hit.r[0] = g0.a; hit.r[1] = g0.b; hit.r[2] = g0.c; hit.r[3] = g0.d;
            hit.r[4] = g1.a; hit.r[5] = g1.b; hit.r[6] = g1.c; hit.r[7] = g1.d;
            kind = static_cast<uint8_t>(kd);
          }
        }
      }
      double hr = 0.0, hi2 = 0.0;
      hit_element<W>(H, J, spos, hit, xrow, lane, s, side, hr, hi2);
      if (valid && !is_diag && !hit.valid) group_element<W>(H, xp, g, hr, hi2);
      // the diagonal as the fused path evaluates it: A + sum_S b_p + sum_{p<q in S} K_pq (+ |z| >= 3 terms)
      if (__any_sync(0xffffffffu, is_diag)) {
        double2 acc = make_double2(0.0, 0.0);
        if (lane == 0) acc.x += side ? H.diag_A1 : H.diag_A0;
        if (lane < s) acc.x += __ldg(H.diag_b + side * nq + spos[lane]);
        const int np = s * (s - 1) / 2;
        for (int pi = lane; pi < np; pi += 32) {
          const int b = static_cast<int>(pair_b(pi)), a = pi - b * (b - 1) / 2;
          acc.x += __ldg(H.diag_K + spos[a] * nq + spos[b]);
        }
        for (uint32_t t2 = lane; t2 < H.n_diag_other; t2 += 32) {
          const uint32_t t = __ldg(H.diag_other + t2);
          int c = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) c += __popcll(xrow.w[w] & __ldg(H.yz + (int64_t)t * W + w));
          const int qt = (__ldg(H.yw + t) + 2 * c) & 3;
          const double cf = __ldg(H.coeff + t);
          if (qt == 0) acc.x += cf;
          else if (qt == 2) acc.x -= cf;
          else if (qt == 1) acc.y += cf;
          else acc.y -= cf;
        }
        acc.x = warp_sum(acc.x);
        acc.y = warp_sum(acc.y);
        if (is_diag) {
          hr = acc.x;
          hi2 = acc.y;
          kind = 5;
        }
      }
      if (valid) {
        out_h[e] = make_double2(hr, hi2);
        out_kind[e] = kind;
      }
    }
  }
}

__global__ void k_check_sorted(const uint32_t* e3, uint64_t n_pairs, int64_t n, int* err) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_pairs;
       e += (uint64_t)gridDim.x * blockDim.x) {
    if (e3[3 * e] >= n || (e > 0 && e3[3 * e] < e3[3 * (e - 1)])) atomicOr(err, kErrBadPair);
  }
}

// per-pair H_{x x'} in reference order, plus the excitation class
template <int W>
__global__ void __launch_bounds__(kThreads)
    k_pair_elements(HamView H, const uint64_t* __restrict__ keys, int64_t n, const uint32_t* __restrict__ e3,
                    uint64_t n_pairs, double2* out_h, uint8_t* out_class, int* err) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_pairs;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = e3[3 * e], j = e3[3 * e + 1], g = e3[3 * e + 2];
    if (x >= n || j >= n || g >= H.n_xy) {
      atomicOr(err, kErrBadPair);
      continue;
    }
    uint64_t xp[W];
#pragma unroll
    for (int w = 0; w < W; ++w) xp[w] = keys[(int64_t)j * W + w];
    double re, im;
    group_element<W>(H, xp, g, re, im);
    out_h[e] = make_double2(re, im);
    if (out_class) out_class[e] = H.xyw[g];
  }
}

// moments (sum w Re E, sum w Im E, sum w^2, sum w, sum w |E|^2) with a
// fixed grid and a fixed reduction tree: deterministic for a given n.
constexpr int kMomentBlocks = 296;

__global__ void __launch_bounds__(kThreads)
    k_moments_partial(const double* __restrict__ lp, double log_norm, const double2* __restrict__ eloc, int64_t n,
                      double* partial, double* weights) {
  double m[5] = {0, 0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double w = exp(lp[i] - log_norm);
    if (weights) weights[i] = w;
    const double2 e = eloc[i];
    m[0] += w * e.x;
    m[1] += w * e.y;
    m[2] += w * w;
    m[3] += w;
    m[4] += w * (e.x * e.x + e.y * e.y);
  }
  __shared__ double sm[kWarps][5];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) m[k] = warp_sum(m[k]);
  if (lane == 0)
    for (int k = 0; k < 5; ++k) sm[wid][k] = m[k];
  __syncthreads();
  if (threadIdx.x < 5) {
    double s = 0;
    for (int w = 0; w < kWarps; ++w) s += sm[w][threadIdx.x];
    partial[blockIdx.x * 5 + threadIdx.x] = s;
  }
}

__global__ void k_moments_final(const double* partial, int n_blocks, double* out) {
  if (threadIdx.x < 5) {
    double s = 0;
    for (int b = 0; b < n_blocks; ++b) s += partial[b * 5 + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// ---------------------------------------------------------------- helpers

template <int W>
void launch_table_build(qvmc_ham_s* h, const uint64_t* keys, int64_t n) {
  // buckets of 4 at load <= 1/4: next power of two >= n buckets
  uint64_t nb = 1;
  while (nb < static_cast<uint64_t>(n)) nb <<= 1;
  nb = std::max<uint64_t>(nb, 64);
  h->tab.ensure(nb * 4 * sizeof(uint64_t));
  h->tab_buckets = nb;
  const int fill_grid = grid_for(h, 4);
  k_fill_u64<<<fill_grid, kThreads, 0, h->stream>>>(h->tab.as<uint64_t>(), nb * 4, kEmpty);
  ck_launch("fill table");
  ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 2, 0, 2 * sizeof(int), h->stream), "memset popcount range");
  TableView T{h->tab.as<uint64_t>(), nb - 1};
  const int grid = static_cast<int>(std::min<int64_t>((n + kThreads - 1) / kThreads + 1, grid_for(h, 8)));
  k_table_build<W><<<grid, kThreads, 0, h->stream>>>(keys, n, h->view.hash_bytes, T, ctl_view(h));
  ck_launch("table build");
}

template <int W, int MODE>
void launch_rows(qvmc_ham_s* h, const uint64_t* keys, int64_t r0, int64_t r1, const RowOut& O) {
  ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 4, 0, 2 * sizeof(int), h->stream), "memset row counter");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows<W, MODE>, kThreads, 0), "occupancy");
  const int64_t warps_needed = r1 - r0;
  const int64_t blocks_needed = (warps_needed + kWarps - 1) / kWarps;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks_needed, grid_for(h, per_sm))));
  TableView T{h->tab.as<uint64_t>(), h->tab_buckets - 1};
  if (r1 > r0) {
    k_rows<W, MODE><<<grid, kThreads, 0, h->stream>>>(h->view, T, keys, r0, r1, ctl_view(h), O);
    ck_launch("row kernel");
  }
}

// How the rows of this call enumerate candidates (needs the popcount range
// the table build just computed: one 8-byte device->host read).
struct RowPlan {
  bool sector = false;
  bool join = false;
  int side = 0;
  int s = 0;
  int key_bits = 0;  // join: bits of the exact bucket rank, ceil(log2 C(n, s - 2))
};

RowPlan plan_from_mm(qvmc_ham_s* h, int64_t n, const int* mm);

RowPlan plan_rows(qvmc_ham_s* h, int64_t n) {
  int mm[2] = {0, 0};
  ck(cudaMemcpyAsync(mm, static_cast<int*>(h->ctl.p) + 2, sizeof(mm), cudaMemcpyDeviceToHost, h->stream), "mm");
  ck(cudaStreamSynchronize(h->stream), "sync");
  const RowPlan P = plan_from_mm(h, n, mm);
  h->plan_ok = true;  // cached for speculative device-memory calls
  h->plan_mm[0] = mm[0];
  h->plan_mm[1] = mm[1];
  h->plan_n = n;
  h->plan_sector = P.sector;
  h->plan_join = P.join;
  h->plan_side = P.side;
  h->plan_s = P.s;
  h->plan_key_bits = P.key_bits;
  return P;
}

RowPlan cached_plan(const qvmc_ham_s* h) {
  RowPlan P;
  P.sector = h->plan_sector;
  P.join = h->plan_join;
  P.side = h->plan_side;
  P.s = h->plan_s;
  P.key_bits = h->plan_key_bits;
  return P;
}

// the speculative plan holds iff the popcount range equals the cached one
__global__ void k_plan_check(const int* __restrict__ mm, int m0, int m1, int* __restrict__ err) {
  if (mm[0] != m0 || mm[1] != m1) atomicOr(err, kErrReplan);
}

RowPlan plan_from_mm(qvmc_ham_s* h, int64_t n, const int* mm) {
  RowPlan P;
  const int pmax = mm[0], pmin = 1024 - mm[1];
  P.side = (pmin <= h->n - pmin) ? 1 : 0;
  P.s = P.side ? pmin : h->n - pmin;
  const bool uniform = n > 0 && pmin == pmax;  // one particle sector
  const uint64_t entries = static_cast<uint64_t>(n) * (P.s * (P.s - 1) / 2);
  P.join = h->use_join && uniform && P.s >= 2 && P.s <= kJoinMaxMinority && entries < (1ull << 31);
  if (P.join) {  // exact bucket keys need C(n, s - 2) < 2^64
    const uint64_t nb = h->binom_host[static_cast<size_t>(h->n) * kBinomK + (P.s - 2)];
    if (nb == ~uint64_t{0}) P.join = false;
    P.key_bits = nb <= 1 ? 1 : 64 - __builtin_clzll(nb - 1);
    if (P.key_bits > 62) P.join = false;  // the distributed build pads with key 1 << key_bits
  }
  // sector structure in use: the join (s <= 32) or the sector candidate lists (s <= 24)
  P.sector = uniform && (P.join || P.s <= kMaxMinorityDev);
  return P;
}

// deletion index: exact keys -> radix sort -> runs -> member array + per-(sample, pair) bucket ranges
template <int W, typename K>
void build_join_index_dist(qvmc_ham_s* h, const uint64_t* keys, int64_t n, const RowPlan& P, bool sym);

template <int W, typename K>
void build_join_index_k(qvmc_ham_s* h, const uint64_t* keys, int64_t n, const RowPlan& P, bool sym) {
  h->dist_active = false;
  if (h->dist_comm && h->dist_comm->world > 1) {
    build_join_index_dist<W, K>(h, keys, n, P, sym);
    return;
  }
  const uint32_t C = static_cast<uint32_t>(P.s * (P.s - 1) / 2);
  const uint64_t E = static_cast<uint64_t>(n) * C;
  h->j_key.ensure(E * sizeof(K) + 16);
  h->j_key2.ensure(E * sizeof(K) + 16);
  h->j_val.ensure(E * 4 + 16);
  h->j_val2.ensure(E * 4 + 16);
  h->j_head.ensure(E * 4 + 16);
  h->j_rid.ensure(E * 4 + 16);
  h->j_lo.ensure(E * 4 + 16);
  h->j_hi.ensure(E * 4 + 16);
  h->j_mem.ensure(E * 8 + 16);
  h->j_rng.ensure(E * 8 + 16);
  const int grid = static_cast<int>(std::min<int64_t>((n + kWarps - 1) / kWarps, grid_for(h, 8)));
  k_join_keys<W, K><<<std::max(grid, 1), kThreads, 0, h->stream>>>(keys, n, h->n, P.side, P.s, h->binom.as<uint64_t>(),
                                                                   h->j_key.as<K>(), h->j_val.as<uint32_t>());
  ck_launch("join keys");
  const int ne = static_cast<int>(E);
  size_t b1 = 0, b2 = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, b1, h->j_key.as<K>(), h->j_key2.as<K>(), h->j_val.as<uint32_t>(),
                                     h->j_val2.as<uint32_t>(), ne, 0, P.key_bits, h->stream),
     "sort size");
  ck(cub::DeviceScan::InclusiveSum(nullptr, b2, h->j_head.as<uint32_t>(), h->j_rid.as<uint32_t>(), ne, h->stream),
     "scan size");
  h->j_tmp.ensure(std::max(b1, b2) + 16);
  ck(cub::DeviceRadixSort::SortPairs(h->j_tmp.p, b1, h->j_key.as<K>(), h->j_key2.as<K>(), h->j_val.as<uint32_t>(),
                                     h->j_val2.as<uint32_t>(), ne, 0, P.key_bits, h->stream),
     "sort");
  ++g_launches;
  const int egrid = static_cast<int>(std::min<uint64_t>((E + kThreads - 1) / kThreads, grid_for(h, 16)));
  k_run_heads<K><<<std::max(egrid, 1), kThreads, 0, h->stream>>>(h->j_key2.as<K>(), E, h->j_head.as<uint32_t>());
  ck_launch("run heads");
  ck(cub::DeviceScan::InclusiveSum(h->j_tmp.p, b2, h->j_head.as<uint32_t>(), h->j_rid.as<uint32_t>(), ne, h->stream),
     "scan");
  ++g_launches;
  k_run_bounds<<<std::max(egrid, 1), kThreads, 0, h->stream>>>(h->j_rid.as<uint32_t>(), E, h->j_lo.as<uint32_t>(),
                                                                h->j_hi.as<uint32_t>());
  ck_launch("run bounds");
  k_join_fill<W><<<std::max(egrid, 1), kThreads, 0, h->stream>>>(h->j_val2.as<uint32_t>(), h->j_rid.as<uint32_t>(), E,
                                                               C, h->j_lo.as<uint32_t>(), h->j_hi.as<uint32_t>(),
                                                               keys, h->n, P.side,
                                                               h->j_mem.as<uint64_t>(), h->j_rng.as<uint2>(),
                                                               sym ? 1 : 0);
  ck_launch("join fill");
}

// Deletion index built across the ranks of a sharded call: every rank computes
// the bucket keys of all entries (cheap), keeps the entries of the buckets it
// owns (a hash of the key; order-preserving selection, so members stay in entry
// order), sorts only those, writes their members and, for every entry of its
// buckets, the bucket range in global positions; one all-gather assembles the
// member array (rank r's slice at r * cap) and one integer all-reduce the
// per-(sample, pair) ranges (each entry is written by exactly one rank). The
// result is the single-GPU index up to where each bucket sits, so the walk, the
// hits and E_loc are bit-identical to it.
template <int W, typename K>
void build_join_index_dist(qvmc_ham_s* h, const uint64_t* keys, int64_t n, const RowPlan& P, bool sym) {
  qvmc_comm_s* cm = h->dist_comm;
  const uint32_t world = static_cast<uint32_t>(cm->world), rank = static_cast<uint32_t>(cm->rank);
  const uint32_t C = static_cast<uint32_t>(P.s * (P.s - 1) / 2);
  const uint64_t E = static_cast<uint64_t>(n) * C;
  const uint64_t cap = std::min<uint64_t>(E, E / world + E / (2 * world) + 4096);  // 1.5x the mean share
  h->j_key.ensure(E * sizeof(K) + 16);
  h->j_key2.ensure(E * sizeof(K) + 16);
  h->j_val.ensure(E * 4 + 16);
  h->j_val2.ensure(E * 4 + 16);
  h->j_head.ensure(cap * 4 + 16);
  h->j_rid.ensure(cap * 4 + 16);
  h->j_lo.ensure(cap * 4 + 16);
  h->j_hi.ensure(cap * 4 + 16);
  h->j_mem.ensure(cap * 8 + 16);
  h->j_memg.ensure(cap * world * 8 + 16);
  h->j_rng.ensure(E * 8 + 16);
  h->j_flags.ensure(E + 16);
  h->j_count.ensure(16);
  const int grid = static_cast<int>(std::min<int64_t>((n + kWarps - 1) / kWarps, grid_for(h, 8)));
  k_join_keys<W, K><<<std::max(grid, 1), kThreads, 0, h->stream>>>(keys, n, h->n, P.side, P.s, h->binom.as<uint64_t>(),
                                                                   h->j_key.as<K>(), h->j_val.as<uint32_t>());
  ck_launch("join keys");
  const int egrid = static_cast<int>(std::min<uint64_t>((E + kThreads - 1) / kThreads, grid_for(h, 16)));
  k_part_flags<K><<<std::max(egrid, 1), kThreads, 0, h->stream>>>(h->j_key.as<K>(), E, world, rank,
                                                                   h->j_flags.as<uint8_t>());
  ck_launch("partition flags");
  const int ne = static_cast<int>(E), nc = static_cast<int>(cap);
  const int key_bits = P.key_bits + 1;  // one more bit: the padding key sorts after every real key
  size_t b0 = 0, b1 = 0, b2 = 0;
  ck(cub::DeviceSelect::Flagged(nullptr, b0, h->j_key.as<K>(), h->j_flags.as<uint8_t>(), h->j_key2.as<K>(),
                                h->j_count.as<uint32_t>(), ne, h->stream), "select size");
  ck(cub::DeviceRadixSort::SortPairs(nullptr, b1, h->j_key2.as<K>(), h->j_key.as<K>(), h->j_val2.as<uint32_t>(),
                                     h->j_val.as<uint32_t>(), nc, 0, key_bits, h->stream), "sort size");
  ck(cub::DeviceScan::InclusiveSum(nullptr, b2, h->j_head.as<uint32_t>(), h->j_rid.as<uint32_t>(), nc, h->stream),
     "scan size");
  h->j_tmp.ensure(std::max({b0, b1, b2}) + 16);
  ck(cub::DeviceSelect::Flagged(h->j_tmp.p, b0, h->j_key.as<K>(), h->j_flags.as<uint8_t>(), h->j_key2.as<K>(),
                                h->j_count.as<uint32_t>(), ne, h->stream), "select keys");
  ck(cub::DeviceSelect::Flagged(h->j_tmp.p, b0, h->j_val.as<uint32_t>(), h->j_flags.as<uint8_t>(),
                                h->j_val2.as<uint32_t>(), h->j_count.as<uint32_t>(), ne, h->stream), "select ids");
  g_launches += 2;
  const int pgrid = static_cast<int>(std::min<uint64_t>((cap + kThreads - 1) / kThreads, grid_for(h, 16)));
  k_pad_slice<K><<<std::max(pgrid, 1), kThreads, 0, h->stream>>>(h->j_key2.as<K>(), h->j_val2.as<uint32_t>(),
                                                                  h->j_count.as<uint32_t>(), cap,
                                                                  static_cast<K>(K{1} << P.key_bits),
                                                                  static_cast<int*>(h->ctl.p));
  ck_launch("pad slice");
  ck(cub::DeviceRadixSort::SortPairs(h->j_tmp.p, b1, h->j_key2.as<K>(), h->j_key.as<K>(), h->j_val2.as<uint32_t>(),
                                     h->j_val.as<uint32_t>(), nc, 0, key_bits, h->stream), "sort slice");
  ++g_launches;
  k_run_heads<K><<<std::max(pgrid, 1), kThreads, 0, h->stream>>>(h->j_key.as<K>(), cap, h->j_head.as<uint32_t>());
  ck_launch("run heads");
  ck(cub::DeviceScan::InclusiveSum(h->j_tmp.p, b2, h->j_head.as<uint32_t>(), h->j_rid.as<uint32_t>(), nc, h->stream),
     "scan");
  ++g_launches;
  k_run_bounds<<<std::max(pgrid, 1), kThreads, 0, h->stream>>>(h->j_rid.as<uint32_t>(), cap, h->j_lo.as<uint32_t>(),
                                                                h->j_hi.as<uint32_t>());
  ck_launch("run bounds");
  ck(cudaMemsetAsync(h->j_rng.p, 0, E * 8, h->stream), "memset ranges");
  k_join_fill<W><<<std::max(pgrid, 1), kThreads, 0, h->stream>>>(
      h->j_val.as<uint32_t>(), h->j_rid.as<uint32_t>(), cap, C, h->j_lo.as<uint32_t>(), h->j_hi.as<uint32_t>(), keys,
      h->n, P.side, h->j_mem.as<uint64_t>(), h->j_rng.as<uint2>(), sym ? 1 : 0, h->j_count.as<uint32_t>(),
      static_cast<uint32_t>(rank * cap));
  ck_launch("join fill (slice)");
  comm_all_gather(cm, h->j_mem.p, h->j_memg.p, cap * 8, h->stream);
  comm_all_reduce_u64(cm, h->j_rng.as<unsigned long long>(), E, h->stream, h->j_rtmp);
  h->dist_active = true;
  h->last.join_mode = 2;
}

template <int W>
void build_join_index(qvmc_ham_s* h, const uint64_t* keys, int64_t n, const RowPlan& P, bool sym = false) {
  h->sym_last = sym;
  const int extra = (h->dist_comm && h->dist_comm->world > 1) ? 1 : 0;  // the slice's padding key
  if (P.key_bits + extra <= 32)
    build_join_index_k<W, uint32_t>(h, keys, n, P, sym);
  else
    build_join_index_k<W, uint64_t>(h, keys, n, P, sym);
}

JoinView join_view(qvmc_ham_s* h, const RowPlan& P) {
  JoinView J{};
  J.C = static_cast<uint32_t>(P.s * (P.s - 1) / 2);
  J.rng = h->j_rng.as<uint2>();
  J.mem = h->dist_active ? h->j_memg.as<uint64_t>() : h->j_mem.as<uint64_t>();
  J.xy_tab = h->p_xy_tab;
  J.xy_mask = h->xy_tab_mask;
  J.rec = h->l_rec.as<uint64_t>();
  J.grec = h->p_grec;
  J.famvi = h->p_famvi;
  J.pbits = h->pbits_P ? h->p_pbits : nullptr;
  J.P = h->pbits_P;
  J.sym = h->sym_last ? 1 : 0;
  return J;
}

// dynamic shared memory of a k_rows_join launch (kModeFused's rings, then one
// bucket-table region per search warp sized by this call's s), with the
// function's limit raised once per device when it exceeds the default
template <int W, int MODE>
size_t join_smem(int s) {
  constexpr bool fused = MODE == kModeFused;
  const int nr = s * (s - 1) / 2;
  const size_t dyn = (fused ? sizeof(FusedSmem) : 0) + static_cast<size_t>(fused ? kFSearch : kWarps) *
                                                          join_range_bytes(nr);
  static size_t set_to[64] = {};
  int dev = 0;
  ck(cudaGetDevice(&dev), "device");
  if (dev >= 0 && dev < 64 && dyn > set_to[dev]) {
    ck(cudaFuncSetAttribute(k_rows_join<W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)),
       "smem attribute");
    set_to[dev] = dyn;
  }
  return dyn;
}

template <int W, int MODE>
void launch_rows_join(qvmc_ham_s* h, const uint64_t* keys, const RowSet& R, const RowPlan& P, const RowOut& O) {
  ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 4, 0, 2 * sizeof(int), h->stream), "memset row counter");
  int per_sm = 0;
  const size_t dyn = join_smem<W, MODE>(P.s);
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows_join<W, MODE>, kThreads, dyn), "occupancy");
  const int64_t blocks_needed = (R.n_rows + kWarps - 1) / kWarps;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks_needed, grid_for(h, per_sm))));
  TableView T{h->tab.as<uint64_t>(), h->tab_buckets - 1};
  if (R.n_rows > 0) {
    k_rows_join<W, MODE><<<grid, kThreads, dyn, h->stream>>>(h->view, T, join_view(h, P), keys, R, P.side, P.s,
                                                           ctl_view(h), O);
    ck_launch("row kernel (join)");
  }
}

// Fused join rows (kModeFused): search warps hand hit chunks to evaluation
// warps through shared memory inside one persistent kernel that writes E_loc
// directly: no hit buffers, nothing to overflow, no host synchronisation.
template <int W>
void run_join_fused(qvmc_ham_s* h, const uint64_t* keys, const RowSet& R, const RowPlan& P, double2* eloc) {
  if (R.n_rows <= 0) return;
  int* ctl = static_cast<int*>(h->ctl.p);
  ck(cudaMemsetAsync(ctl + 4, 0, 2 * sizeof(int), h->stream), "memset row counter");
  int per_sm = 0;
  const size_t dyn = join_smem<W, kModeFused>(P.s);
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows_join<W, kModeFused>, kFThreads, dyn), "occupancy");
  const int64_t blocks_needed = (R.n_rows + kFSearch - 1) / kFSearch;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks_needed, grid_for(h, per_sm))));
  RowOut O{};
  O.eloc = eloc;
  O.exp_flag = ctl + 14;
  TableView T{h->tab.as<uint64_t>(), h->tab_buckets - 1};
  if (!h->ev_f[0]) {
    ck(cudaEventCreate(&h->ev_f[0]), "event create");
    ck(cudaEventCreate(&h->ev_f[1]), "event create");
  }
  ck(cudaEventRecord(h->ev_f[0], h->stream), "event");
  k_rows_join<W, kModeFused><<<grid, kFThreads, dyn, h->stream>>>(h->view, T, join_view(h, P), keys, R, P.side,
                                                                  P.s, ctl_view(h), O);
  ck_launch("row kernel (join, fused search + evaluation)");
  ck(cudaEventRecord(h->ev_f[1], h->stream), "event");
  h->timed_f = true;
}

// Pipelined split evaluation: rows in NB batches, the search of batch b+1
// (stream A) overlaps the evaluation of batch b (stream B), two buffer sets in
// turn. The search is issue-bound and the evaluation latency-bound, so the
// two fill each other's idle issue slots when they share SMs. Overflow of a
// batch's buffers is detected after the last batch (no mid-call sync); the
// whole pipeline then reruns with larger buffers.
template <int W>
bool run_join_pipelined(qvmc_ham_s* h, const uint64_t* keys, int64_t n_all, const RowSet& R, const RowPlan& P,
                        double2* eloc, bool spec = false) {
  // symmetric index (h->sym_last): mirrored contributions accumulate exactly in s_fix; the row
  // batches are contiguous sorted positions evaluated in order, so a row's mirrored sums from
  // rows x < y are complete when its own batch has been evaluated
  unsigned long long* fix = nullptr;
  if (h->sym_last) {
    h->s_fix.ensure(static_cast<size_t>(n_all) * 32 + 16);
    fix = h->s_fix.as<unsigned long long>();
  }
  const int64_t rows = R.n_rows;
  if (rows <= 0) return false;
  constexpr uint64_t kBatchHits = 1ull << 31;
  const uint64_t per_row = std::max<uint64_t>(h->hits_per_row, 64);
  const int64_t nb_min = static_cast<int64_t>((static_cast<uint64_t>(rows) * per_row + kBatchHits - 1) / kBatchHits);
  const int64_t NB = std::min<int64_t>(rows, std::max<int64_t>(h->pipe_batches, nb_min));
  const int64_t batch = (rows + NB - 1) / NB;
  if (h->p_hit_cap == 0) {
    h->p_hit_cap = std::min<uint64_t>(static_cast<uint64_t>(batch) * per_row * 5 / 4 + (1u << 16), 0xFFFFFFFFull);
    h->p_chunk_cap = h->p_hit_cap / 32 + static_cast<uint64_t>(batch) + 1024;
  }
  // per-row outputs are indexed by caller row - R.out_base: a strided sharded walk spans every row
  const int64_t span = h->walk_world > 1 ? n_all : rows;
  h->s_row_last.ensure(span * 4 + 16);
  h->s_base.ensure(span * 16 + 16);
  h->s_rowpos.ensure(static_cast<size_t>(n_all) * 32 + 16);
  if (!h->side) {
    ck(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking), "stream create");
    for (auto& e : h->ev_p) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
  }
  if (static_cast<int64_t>(h->log_cap) < NB) {
    if (h->log_host) cudaFreeHost(h->log_host);
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h->log_host), NB * 2 * sizeof(unsigned long long), cudaHostAllocDefault),
       "pinned log");
    h->log_cap = static_cast<uint64_t>(NB);
  }
  int* ctl = static_cast<int*>(h->ctl.p);
  cudaStream_t A = h->stream, B = h->side;
  cudaEvent_t ev_start = h->ev_p[0], ev_join = h->ev_p[1], ev_s[2] = {h->ev_p[2], h->ev_p[3]},
              ev_e[2] = {h->ev_p[4], h->ev_p[5]};
  while (static_cast<int64_t>(h->ev_b.size()) < 4 * NB) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event create");
    h->ev_b.push_back(e);
  }
  h->timed_b = 0;
  for (int attempt = 0;; ++attempt) {
    if (fix) ck(cudaMemsetAsync(fix, 0, static_cast<size_t>(n_all) * 32, h->stream), "memset fix");
    for (int k = 0; k < 2; ++k) {
      h->p_hy[k].ensure(h->p_hit_cap * 4 + 16);
      h->p_hg[k].ensure(h->p_hit_cap * 4 + 16);
      h->p_hk[k].ensure(h->p_hit_cap * 4 + 16);
      h->p_chunk[k].ensure(h->p_chunk_cap * 16 + 16);
      h->p_part[k].ensure(h->p_chunk_cap * 16 + 16);
    }
    int per_sm_s = 0, per_sm_e = 0;
    const size_t dyn_s = join_smem<W, kModeHits>(P.s);
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, k_rows_join<W, kModeHits>, kThreads, dyn_s),
       "occupancy");
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_e, k_eval_chunks<W>, kThreads, 0), "occupancy");
    if (h->pipe_search_blocks > 0) per_sm_s = std::min(per_sm_s, h->pipe_search_blocks);
    if (h->pipe_eval_blocks > 0) per_sm_e = std::min(per_sm_e, h->pipe_eval_blocks);
    ck(cudaEventRecord(ev_start, A), "event");
    ck(cudaStreamWaitEvent(B, ev_start, 0), "wait");
    TableView T{h->tab.as<uint64_t>(), h->tab_buckets - 1};
    for (int64_t b = 0; b < NB; ++b) {
      const int k = static_cast<int>(b & 1);
      RowSet Rb = R;
      Rb.n_rows = std::min<int64_t>(batch, rows - b * batch);
      if (Rb.n_rows <= 0) {
        h->log_host[2 * b] = h->log_host[2 * b + 1] = 0;
        continue;
      }
      if (R.list) Rb.list = R.list + b * batch;
      else Rb.base = R.base + b * batch;
      int* cur = ctl + 16 + 4 * k;  // this set's hit / chunk cursors (u64 each)
      if (b >= 2) ck(cudaStreamWaitEvent(A, ev_e[k], 0), "wait");
      ck(cudaMemsetAsync(ctl + 4, 0, 2 * sizeof(int), A), "memset row counter");
      ck(cudaMemsetAsync(cur, 0, 4 * sizeof(int), A), "memset cursors");
      RowOut O{};
      O.hy = h->p_hy[k].as<uint32_t>();
      O.hg = h->p_hg[k].as<uint32_t>();
      O.hk = h->p_hk[k].as<uint32_t>();
      O.chunk = h->p_chunk[k].as<uint4>();
      O.row_last = h->s_row_last.as<uint32_t>();
      O.base = h->s_base.as<double2>();
      O.hit_cursor = reinterpret_cast<unsigned long long*>(cur);
      O.chunk_cursor = reinterpret_cast<unsigned long long*>(cur + 2);
      O.hit_cap = h->p_hit_cap;
      O.chunk_cap = h->p_chunk_cap;
      O.rowpos = h->s_rowpos.as<uint8_t>();
      const int grid_s = static_cast<int>(
          std::max<int64_t>(1, std::min<int64_t>((Rb.n_rows + kWarps - 1) / kWarps, grid_for(h, per_sm_s))));
      ck(cudaEventRecord(h->ev_b[4 * b], A), "event");
      k_rows_join<W, kModeHits><<<grid_s, kThreads, dyn_s, A>>>(h->view, T, join_view(h, P), keys, Rb, P.side, P.s,
                                                            ctl_view(h), O);
      ck_launch("row kernel (join search)");
      ck(cudaEventRecord(h->ev_b[4 * b + 1], A), "event");
      ck(cudaMemcpyAsync(h->log_host + 2 * b, cur, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, A),
         "D2H cursors");
      ck(cudaEventRecord(ev_s[k], A), "event");
      ck(cudaStreamWaitEvent(B, ev_s[k], 0), "wait");
      ck(cudaEventRecord(h->ev_b[4 * b + 2], B), "event");
      k_eval_chunks<W><<<grid_for(h, per_sm_e), kThreads, 0, B>>>(
          h->view, join_view(h, P), keys, h->p_chunk[k].as<uint4>(), reinterpret_cast<unsigned long long*>(cur + 2),
          h->p_hy[k].as<uint32_t>(), h->p_hg[k].as<uint32_t>(), h->p_hk[k].as<uint32_t>(), P.side, P.s, ctl + 14,
          h->s_rowpos.as<uint8_t>(), h->p_part[k].as<double2>(), h->p_chunk_cap, fix, ctl);
      ck_launch("eval chunks");
      ck(cudaEventRecord(h->ev_b[4 * b + 3], B), "event");
      const int fgrid = static_cast<int>(std::min<int64_t>((Rb.n_rows + kThreads - 1) / kThreads, grid_for(h, 8)));
      k_finalize_rows<<<std::max(fgrid, 1), kThreads, 0, B>>>(h->s_row_last.as<uint32_t>(), h->p_chunk[k].as<uint4>(),
                                                              h->p_part[k].as<double2>(), h->s_base.as<double2>(), Rb,
                                                              eloc, h->shard_sym ? nullptr : fix);
      ck_launch("finalize rows");
      ck(cudaEventRecord(ev_e[k], B), "event");
    }
    ck(cudaEventRecord(ev_join, B), "event");
    ck(cudaStreamWaitEvent(A, ev_join, 0), "wait");
    if (spec) {  // no host round trip: an overflow (kErrHitOverflow) is handled by qvmc_cuda_synchronize
      h->timed_b = (rows + batch - 1) / batch;
      h->pend_nb = NB;
      return false;
    }
    ck(cudaStreamSynchronize(A), "sync");
    if (fix) {  // a mirrored contribution out of the fixed-point range: the caller redoes the call unpaired
      int err = 0;
      ck(cudaMemcpy(&err, ctl, sizeof(int), cudaMemcpyDeviceToHost), "read err");
      if (err & kErrFixRange) {
        err &= ~kErrFixRange;
        ck(cudaMemcpy(ctl, &err, sizeof(int), cudaMemcpyHostToDevice), "reset err");
        return true;
      }
    }
    uint64_t need_h = 0, need_c = 0, hits = 0;
    for (int64_t b = 0; b < NB; ++b) {
      need_h = std::max<uint64_t>(need_h, h->log_host[2 * b]);
      need_c = std::max<uint64_t>(need_c, h->log_host[2 * b + 1]);
      hits += h->log_host[2 * b];
    }
    h->timed_b = (rows + batch - 1) / batch;  // non-empty batches (each recorded its four events)
    if (need_h <= h->p_hit_cap && need_c <= h->p_chunk_cap) {
      h->hits_per_row = std::max<uint64_t>(h->hits_per_row, hits / static_cast<uint64_t>(rows) + 1);
      break;
    }
    if (fix) ck(cudaMemsetAsync(fix, 0, static_cast<size_t>(n_all) * 32, h->stream), "memset fix");
    if (attempt >= 3 || h->p_hit_cap >= 0xFFFFFFFFull) fail(QVMC_ERR_RUNTIME, "join hit buffers keep overflowing");
    h->p_hit_cap = std::min<uint64_t>(std::max<uint64_t>(h->p_hit_cap, need_h + need_h / 4 + 1024), 0xFFFFFFFFull);
    h->p_chunk_cap = std::max<uint64_t>(h->p_chunk_cap, need_c + need_c / 4 + 1024);
    int err = 0;  // rerun from scratch: counters of the overflowed attempt dropped
    ck(cudaMemcpy(&err, ctl, sizeof(int), cudaMemcpyDeviceToHost), "read err");
    err &= ~kErrHitOverflow;
    ck(cudaMemcpy(ctl, &err, sizeof(int), cudaMemcpyHostToDevice), "reset overflow");
    ck(cudaMemset(ctl + 6, 0, 4 * sizeof(int)), "reset stats");
  }
  return false;
}

template <int W, int MODE>
void run_rows(qvmc_ham_s* h, const uint64_t* keys, int64_t r0, int64_t r1, const RowPlan& P, const RowOut& O) {
  if (P.join)
    launch_rows_join<W, MODE>(h, keys, RowSet{r1 - r0, r0, nullptr, nullptr, r0}, P, O);
  else
    launch_rows<W, MODE>(h, keys, r0, r1, O);
}

// Join mode of the fused call: sort the sample set by minority orbitals
// (locality), rebuild the index on the sorted copy, process rows in that
// order. Returns the row set; keys/la/ph are redirected to the sorted copies.
template <int W>
RowSet sort_for_locality(qvmc_ham_s* h, const uint64_t*& keys, int64_t n, int64_t r0, int64_t r1,
                         const RowPlan& P) {
  h->l_key.ensure(n * 8 + 16);
  h->l_key2.ensure(n * 8 + 16);
  h->l_idx.ensure(n * 4 + 16);
  h->l_perm.ensure(n * 4 + 16);
  h->l_keys.ensure(n * 8 * W + 16);
  h->l_rec.ensure(n * 32 + 32);
  const int grid = static_cast<int>(std::min<int64_t>((n + kThreads - 1) / kThreads, grid_for(h, 8)));
  k_locality_keys<W><<<std::max(grid, 1), kThreads, 0, h->stream>>>(keys, n, h->n, P.side, h->l_key.as<uint64_t>(),
                                                                    h->l_idx.as<uint32_t>());
  ck_launch("locality keys");
  size_t bytes = 0;
  const int ni = static_cast<int>(n);
  ck(cub::DeviceRadixSort::SortPairs(nullptr, bytes, h->l_key.as<uint64_t>(), h->l_key2.as<uint64_t>(),
                                     h->l_idx.as<uint32_t>(), h->l_perm.as<uint32_t>(), ni, 0, 64, h->stream),
     "sort size");
  h->j_tmp.ensure(bytes + 16);
  ck(cub::DeviceRadixSort::SortPairs(h->j_tmp.p, bytes, h->l_key.as<uint64_t>(), h->l_key2.as<uint64_t>(),
                                     h->l_idx.as<uint32_t>(), h->l_perm.as<uint32_t>(), ni, 0, 64, h->stream),
     "sort");
  ++g_launches;
  k_gather_keys<W><<<std::max(grid, 1), kThreads, 0, h->stream>>>(h->l_perm.as<uint32_t>(), n, keys,
                                                                  h->l_keys.as<uint64_t>());
  ck_launch("gather sorted keys");
  keys = h->l_keys.as<uint64_t>();
  RowSet R{n, 0, nullptr, h->l_perm.as<uint32_t>(), r0};
  if (h->walk_world > 1) {  // sharded call, strided walk: every world-th sorted position (balanced
    // whatever the caller's sample order: neighbours in locality order cost about the same)
    const int64_t nr = n > h->walk_rank ? (n - h->walk_rank + h->walk_world - 1) / h->walk_world : 0;
    h->l_list.ensure(std::max<int64_t>(nr, 1) * 4 + 16);
    const int sg = static_cast<int>(std::min<int64_t>((std::max<int64_t>(nr, 1) + kThreads - 1) / kThreads,
                                                      grid_for(h, 8)));
    k_strided_rows<<<sg, kThreads, 0, h->stream>>>(h->l_list.as<uint32_t>(), nr,
                                                   static_cast<uint32_t>(h->walk_rank),
                                                   static_cast<uint32_t>(h->walk_world));
    ck_launch("strided rows");
    R.list = h->l_list.as<uint32_t>();
    R.n_rows = nr;
  } else if (r0 != 0 || r1 != n) {  // a row shard: the sorted positions of its rows
    h->l_flags.ensure(n + 16);
    h->l_list.ensure(n * 4 + 16);
    h->l_nsel.ensure(16);
    k_flag_rows<<<std::max(grid, 1), kThreads, 0, h->stream>>>(h->l_perm.as<uint32_t>(), n, r0, r1,
                                                               h->l_flags.as<uint8_t>());
    ck_launch("flag rows");
    bytes = 0;
    thrust::counting_iterator<uint32_t> it(0);
    ck(cub::DeviceSelect::Flagged(nullptr, bytes, it, h->l_flags.as<uint8_t>(), h->l_list.as<uint32_t>(),
                                  h->l_nsel.as<int>(), ni, h->stream),
       "select size");
    h->j_tmp.ensure(bytes + 16);
    ck(cub::DeviceSelect::Flagged(h->j_tmp.p, bytes, it, h->l_flags.as<uint8_t>(), h->l_list.as<uint32_t>(),
                                  h->l_nsel.as<int>(), ni, h->stream),
       "select");
    ++g_launches;
    R.list = h->l_list.as<uint32_t>();
    R.n_rows = r1 - r0;
  }
  return R;
}

// the sample records in the order sort_for_locality chose (needs the amplitudes)
void gather_records(qvmc_ham_s* h, const double* la, const double* ph, int64_t n) {
  const int grid = static_cast<int>(std::min<int64_t>((n + kThreads - 1) / kThreads, grid_for(h, 8)));
  ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 14, 0, sizeof(int), h->stream), "memset exp flag");
  k_gather_records<<<std::max(grid, 1), kThreads, 0, h->stream>>>(h->l_perm.as<uint32_t>(), n, la, ph,
                                                                   h->l_rec.as<double>(),
                                                                   static_cast<int*>(h->ctl.p) + 14);
  ck_launch("gather sorted records");
}

void note_plan(qvmc_ham_s* h, const RowPlan& P) {
  h->last.sector_mode = P.sector ? 1 : 0;
  h->last.sector_side = P.side;
  h->last.minority_count = P.s;
  h->last.join_mode = P.join ? 1 : 0;
}

int read_err_and_reset(qvmc_ham_s* h) {
  int err = 0;
  ck(cudaMemcpyAsync(&err, h->ctl.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream), "read err");
  ck(cudaStreamSynchronize(h->stream), "sync");
  if (err) ck(cudaMemsetAsync(h->ctl.p, 0, sizeof(int), h->stream), "reset err");
  return err;
}

void raise_device_err(int err) {
  if (err & kErrSliceOverflow)
    fail(QVMC_ERR_RUNTIME, "distributed deletion index: a rank's share exceeded its capacity (QVMC_DIST_INDEX=0)");
  if (err & kErrDuplicate) fail(QVMC_ERR_INVALID_ARGUMENT, "sample set contains duplicate basis vectors");
  if (err & kErrBadPair) fail(QVMC_ERR_INVALID_ARGUMENT, "pair entry out of range or not in canonical order");
  if (err & kErrZeroAmp) fail(QVMC_ERR_LOGIC, "local_energies: sampled state has zero amplitude");
}

void resolve_pending(qvmc_ham_s* h);

void finish(qvmc_ham_s* h) {
  if (h->pending) resolve_pending(h);
  const int err = read_err_and_reset(h);
  if (err) raise_device_err(err);
}

// stage a host array into a workspace buffer (or pass a device pointer through)
template <typename T>
const T* stage(qvmc_ham_s* h, DBuf& buf, const T* src, size_t count, int mem) {
  if (mem == QVMC_MEM_DEVICE) return src;
  buf.ensure(std::max<size_t>(count * sizeof(T), 16));
  if (count) ck(cudaMemcpyAsync(buf.p, src, count * sizeof(T), cudaMemcpyHostToDevice, h->stream), "H2D");
  return buf.as<T>();
}

void check_mem(int mem) {
  if (mem != QVMC_MEM_HOST && mem != QVMC_MEM_DEVICE) fail(QVMC_ERR_INVALID_ARGUMENT, "unknown memory kind");
}

#define DISPATCH_W(W_, ...)                                       \
  switch (W_) {                                                   \
    case 1: { constexpr int WW = 1; __VA_ARGS__; break; }         \
    case 2: { constexpr int WW = 2; __VA_ARGS__; break; }         \
    case 3: { constexpr int WW = 3; __VA_ARGS__; break; }         \
    case 4: { constexpr int WW = 4; __VA_ARGS__; break; }         \
    default: fail(QVMC_ERR_INVALID_ARGUMENT, "unsupported word count"); \
  }

void compute_moments(qvmc_ham_s* h, const double* lp, double log_norm, const double2* eloc, int64_t n,
                     double* out_dev, double* weights_dev) {
  h->partials.ensure(kMomentBlocks * 5 * sizeof(double));
  k_moments_partial<<<kMomentBlocks, kThreads, 0, h->stream>>>(lp, log_norm, eloc, n, h->partials.as<double>(),
                                                               weights_dev);
  ck_launch("moments partial");
  k_moments_final<<<1, 32, 0, h->stream>>>(h->partials.as<double>(), kMomentBlocks, out_dev);
  ck_launch("moments final");
}

// Check a speculative call (synchronises): if its cached plan did not hold or a hit
// buffer overflowed, grow the buffers / drop the plan and rerun it synchronously from
// the kept arguments (the caller keeps them valid until qvmc_cuda_synchronize).
void resolve_pending(qvmc_ham_s* h) {
  h->pending = false;
  ck(cudaStreamSynchronize(h->pend_stream), "sync");  // the stream may have been switched since the call
  cudaStream_t cur = h->stream;
  h->stream = h->pend_stream;  // a rerun goes to the same stream
  int err = 0;
  ck(cudaMemcpy(&err, h->ctl.p, sizeof(int), cudaMemcpyDeviceToHost), "read err");
  uint64_t need_h = 0, need_c = 0, hits = 0;
  for (int64_t b = 0; b < h->pend_nb && h->log_host; ++b) {
    need_h = std::max<uint64_t>(need_h, h->log_host[2 * b]);
    need_c = std::max<uint64_t>(need_c, h->log_host[2 * b + 1]);
    hits += h->log_host[2 * b];
  }
  h->pend_nb = 0;
  if (err & kErrFixRange) h->sym_off_once = true;
  if (!(err & (kErrReplan | kErrHitOverflow | kErrFixRange))) {
    h->stream = cur;
    const int64_t rows = h->pend.r1 - h->pend.r0;
    if (rows > 0 && hits) h->hits_per_row = std::max<uint64_t>(h->hits_per_row, hits / static_cast<uint64_t>(rows) + 1);
    return;  // other device errors are reported by finish()
  }
  if (err & kErrHitOverflow) {
    h->p_hit_cap = std::min<uint64_t>(std::max<uint64_t>(h->p_hit_cap, need_h + need_h / 4 + 1024), 0xFFFFFFFFull);
    h->p_chunk_cap = std::max<uint64_t>(h->p_chunk_cap, need_c + need_c / 4 + 1024);
  }
  h->plan_ok = false;  // the rerun plans synchronously (and re-caches the plan)
  ck(cudaMemset(h->ctl.p, 0, sizeof(int)), "reset err");
  const auto a = h->pend;
  const int st = qvmc_cuda_eloc_fused(h, a.n_unq, a.keys, a.la, a.ph, a.lp, a.log_norm, a.r0, a.r1, a.eloc,
                                      a.moments, QVMC_MEM_DEVICE);
  ck(cudaStreamSynchronize(h->stream), "sync");
  h->stream = cur;
  if (st != QVMC_OK) fail(st, g_error);
}

void record_stats(qvmc_ham_s* h, int64_t rows) {
  h->timed = false;
  h->timed_b = 0;
  h->timed_f = false;
  h->last = qvmc_stats{};
  h->last.rows = static_cast<uint64_t>(rows);
  h->last.terms_equivalent = static_cast<uint64_t>(rows) * h->n_xy;
}

}  // namespace

// ================================================================ C ABI

extern "C" {

const char* qvmc_cuda_last_error(void) { return g_error.c_str(); }
uint64_t qvmc_cuda_launch_count(void) { return g_launches.load(); }

int qvmc_index_build(int n_qubits, int n_words, int64_t n_raw, const double* coeff, const uint64_t* x_words,
                     const uint64_t* y_words, const uint64_t* z_words, qvmc_index_t* out) {
  return guarded([&] {
    if (!out || (n_raw > 0 && (!coeff || !x_words || !y_words || !z_words)))
      fail(QVMC_ERR_INVALID_ARGUMENT, "null argument");
    auto box = std::make_unique<qvmc_index_s>();
    box->idx = index_from_terms(n_qubits, n_words, n_raw, coeff, x_words, y_words, z_words);
    *out = box.release();
  });
}

int qvmc_index_info(qvmc_index_t idx, int* n_qubits, uint64_t* n_terms, uint32_t* n_xy, int64_t* diag) {
  return guarded([&] {
    if (!idx) fail(QVMC_ERR_INVALID_ARGUMENT, "null index");
    if (n_qubits) *n_qubits = idx->idx.n_qubits;
    if (n_terms) *n_terms = idx->idx.n_terms();
    if (n_xy) *n_xy = idx->idx.n_xy();
    if (diag) *diag = idx->idx.diag;
  });
}

int qvmc_index_export(qvmc_index_t idx, uint64_t* xy_words, uint64_t* group_offsets, double* coeff,
                      uint64_t* yz_words, uint8_t* y_weight, uint64_t* x_words, uint64_t* y_words,
                      uint64_t* z_words) {
  return guarded([&] {
    if (!idx) fail(QVMC_ERR_INVALID_ARGUMENT, "null index");
    const HostIndex& h = idx->idx;
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(xy_words, h.xy);
    cp(group_offsets, h.offsets);
    cp(coeff, h.coeff);
    cp(yz_words, h.yz);
    cp(y_weight, h.y_weight);
    cp(x_words, h.x);
    cp(y_words, h.y);
    cp(z_words, h.z);
  });
}

void qvmc_index_destroy(qvmc_index_t idx) { delete idx; }

int qvmc_index_plan_summary(qvmc_index_t idx, qvmc_plan_summary* out) {
  return guarded([&] {
    if (!idx || !out) fail(QVMC_ERR_INVALID_ARGUMENT, "null argument");
    const HostIndex& hi = idx->idx;
    const DevicePlan p = plan_device(hi);
    qvmc_plan_summary r{};
    for (uint32_t g = 0; g < hi.n_xy(); ++g) {
      if (static_cast<int64_t>(g) == hi.diag) continue;
      const uint64_t kind = p.grec[static_cast<size_t>(g) * kGrecWordsHost] & 3;
      (kind == 0 ? r.kind_a : kind == 1 ? r.kind_b : kind == 2 ? r.kind_c : r.kind_d) += 1;
      if (p.xy_weight[g] == 2) ++r.singles;
      if (p.xy_weight[g] == 4) ++r.doubles;
    }
    for (uint32_t w : p.pbits) r.bitmap_bits += static_cast<uint64_t>(std::popcount(w));
    r.xy_tab_buckets = p.xy_tab_mask + 1;
    *out = r;
  });
}

int qvmc_cuda_ham_create(int n_qubits, int n_words, uint32_t n_xy, const uint64_t* xy_words,
                         const uint64_t* group_offsets, uint64_t n_terms, const double* coeff,
                         const uint64_t* yz_words, const uint8_t* y_weight, int64_t diag_xy, int device,
                         qvmc_ham_t* out) {
  return guarded([&] {
    if (!out) fail(QVMC_ERR_INVALID_ARGUMENT, "null output handle");
    if (n_qubits < 1 || n_qubits > 256 || n_words != (n_qubits + 63) / 64)
      fail(QVMC_ERR_INVALID_ARGUMENT, "qubit count out of range or n_words != ceil(N/64)");
    if (n_xy > 0 && (!xy_words || !group_offsets)) fail(QVMC_ERR_INVALID_ARGUMENT, "null xy arrays");
    if (n_terms > 0 && (!coeff || !yz_words || !y_weight)) fail(QVMC_ERR_INVALID_ARGUMENT, "null term arrays");
    if (diag_xy >= static_cast<int64_t>(n_xy)) fail(QVMC_ERR_INVALID_ARGUMENT, "diag_xy out of range");
    HostIndex hi;
    hi.n_qubits = n_qubits;
    hi.n_words = n_words;
    hi.xy.assign(xy_words, xy_words + static_cast<size_t>(n_xy) * n_words);
    hi.offsets.assign(group_offsets, group_offsets + n_xy + 1);
    if (n_xy == 0) hi.offsets.assign(1, 0);
    if (hi.offsets.back() != n_terms || hi.offsets.front() != 0)
      fail(QVMC_ERR_INVALID_ARGUMENT, "group offsets do not span the terms");
    for (uint32_t g = 0; g < n_xy; ++g)
      if (hi.offsets[g] > hi.offsets[g + 1]) fail(QVMC_ERR_INVALID_ARGUMENT, "group offsets not monotone");
    hi.coeff.assign(coeff, coeff + n_terms);
    hi.yz.assign(yz_words, yz_words + n_terms * n_words);
    hi.y_weight.assign(y_weight, y_weight + n_terms);
    hi.diag = diag_xy;

    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) fail(QVMC_ERR_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= n_dev) fail(QVMC_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    DeviceGuard dg(device);
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) fail(QVMC_ERR_NO_DEVICE, "libqvmc_cuda is built for sm_100a (B200) only");

    const DevicePlan p = plan_device(hi);
    auto h = std::make_unique<qvmc_ham_s>();
    h->device = device;
    h->n = n_qubits;
    h->W = n_words;
    h->n_xy = n_xy;
    h->diag = diag_xy;
    h->n_terms = n_terms;
    h->sms = prop.multiProcessorCount;
    ck(cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking), "stream create");
    h->stream = h->own;
    for (auto& e : h->ev) ck(cudaEventCreate(&e), "event create");
    upload(h->xy, hi.xy);
    upload(h->xy_hash, p.xy_hash);
    upload(h->goff, p.offsets32);
    upload(h->coeff, hi.coeff);
    upload(h->yz, hi.yz);
    upload(h->yw, hi.y_weight);
    upload(h->xyw, p.xy_weight);
    upload(h->gen_hash, p.gen_hash);
    upload(h->gen_g, p.gen_g);
    upload(h->lst_off, p.lst_off);
    upload(h->lst_hash, p.lst_hash);
    upload(h->lst_g, p.lst_g);
    upload(h->res_g, p.res_g);
    upload(h->diag_b, p.diag_b);
    upload(h->diag_K, p.diag_K);
    upload(h->diag_other, p.diag_other);
    upload(h->hash_bytes, p.hash_bytes);

    upload(h->comp_of, p.comp_of);
    upload(h->fam_off, p.fam_off);
    upload(h->fam_B, p.fam_B);
    upload(h->fam_q, p.fam_q);
    upload(h->fam_u, p.fam_u);
    upload(h->fam_V, p.fam_V);
    upload(h->fam_v, p.fam_v);
    upload(h->ginfo, p.ginfo);
    upload(h->trec, p.trec);
    upload(h->famrec, p.famrec);
    {  // the join's hot tables in one arena
      size_t at = 0;
      auto place = [&](size_t bytes) {
        const size_t o = at;
        at = (at + std::max<size_t>(bytes, 16) + 255) & ~size_t{255};
        return o;
      };
      const size_t o_grec = place(p.grec.size() * 8), o_famvi = place(p.famvi.size() * 8),
                   o_pbits = place(p.pbits.size() * 4), o_tab = place(p.xy_tab.size() * 8);
      h->hot.ensure(at);
      h->hot_bytes = at;
      char* base = h->hot.as<char>();
      auto put = [&](size_t o, const void* src, size_t bytes) {
        if (bytes) ck(cudaMemcpy(base + o, src, bytes, cudaMemcpyHostToDevice), "upload hot");
      };
      put(o_grec, p.grec.data(), p.grec.size() * 8);
      put(o_famvi, p.famvi.data(), p.famvi.size() * 8);
      put(o_pbits, p.pbits.data(), p.pbits.size() * 4);
      put(o_tab, p.xy_tab.data(), p.xy_tab.size() * 8);
      h->p_grec = reinterpret_cast<uint64_t*>(base + o_grec);
      h->p_famvi = reinterpret_cast<double*>(base + o_famvi);
      h->p_pbits = reinterpret_cast<uint32_t*>(base + o_pbits);
      h->p_xy_tab = reinterpret_cast<uint64_t*>(base + o_tab);
      // (a persisting L2 access-policy window over this arena measured slower:
      // it takes L2 from the per-call index sort; profiles/r01_tuning_log.txt)
    }
    h->pbits_P = p.pbits_P;
    h->binom_host = binomial_table();
    upload(h->binom, h->binom_host);
    h->xy_tab_mask = p.xy_tab_mask;
    upload(h->codes, std::vector<uint64_t>(qubit_codes(), qubit_codes() + 256));
    {
      std::vector<uint32_t> gk(std::max<uint32_t>(n_xy, 1), 0xFFFFFFFFu);
      for (uint32_t g = 0; g < n_xy; ++g)
        if (p.xy_weight[g] == 2 || p.xy_weight[g] == 4) gk[g] = xy_position_key(&hi.xy[static_cast<size_t>(g) * n_words], n_words);
      upload(h->gkey, gk);
    }
    if (const char* e = std::getenv("QVMC_JOIN")) h->use_join = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_FUSED")) h->fused = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_SYMMETRIC")) h->sym = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_DIST_INDEX")) h->dist_index = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_STRIDED_SHARDS")) h->strided_shards = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_SPECULATE")) h->no_spec = std::atoi(e) == 0;  // opt-in
    if (const char* e = std::getenv("QVMC_PIPE_BATCHES")) h->pipe_batches = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("QVMC_PIPE_SEARCH_BLOCKS")) h->pipe_search_blocks = std::atoi(e);
    if (const char* e = std::getenv("QVMC_PIPE_EVAL_BLOCKS")) h->pipe_eval_blocks = std::atoi(e);
    if (const char* e = std::getenv("QVMC_HIT_CAP")) {  // test hook: a small first capacity exercises the regrow path
      h->p_hit_cap = std::strtoull(e, nullptr, 10);
      h->p_chunk_cap = h->p_hit_cap / 8 + 64;
    }
    h->ctl.ensure(kCtlInts * sizeof(int) * 2);
    ck(cudaMemset(h->ctl.p, 0, kCtlInts * sizeof(int) * 2), "memset ctl");

    HamView& v = h->view;
    v.n = n_qubits;
    v.n_xy = n_xy;
    v.diag = static_cast<int32_t>(diag_xy);
    v.xy = h->xy.as<uint64_t>();
    v.xy_hash = h->xy_hash.as<uint64_t>();
    v.goff = h->goff.as<uint32_t>();
    v.coeff = h->coeff.as<double>();
    v.yz = h->yz.as<uint64_t>();
    v.yw = h->yw.as<uint8_t>();
    v.xyw = h->xyw.as<uint8_t>();
    v.gen_hash = h->gen_hash.as<uint64_t>();
    v.gen_g = h->gen_g.as<uint32_t>();
    v.n_gen = static_cast<uint32_t>(p.gen_g.size());
    v.lst_off = h->lst_off.as<uint32_t>();
    v.lst_hash = h->lst_hash.as<uint64_t>();
    v.lst_g = h->lst_g.as<uint32_t>();
    v.res_g = h->res_g.as<uint32_t>();
    v.n_res = static_cast<uint32_t>(p.res_g.size());
    v.diag_quad = p.diag_quad ? 1 : 0;
    v.diag_A0 = p.diag_A[0];
    v.diag_A1 = p.diag_A[1];
    v.diag_b = h->diag_b.as<double>();
    v.diag_K = h->diag_K.as<double>();
    v.diag_other = h->diag_other.as<uint32_t>();
    v.n_diag_other = static_cast<uint32_t>(p.diag_other.size());
    v.hash_bytes = h->hash_bytes.as<uint64_t>();
    v.comp_of = h->comp_of.as<int32_t>();
    v.fam_off = h->fam_off.as<uint32_t>();
    v.fam_B = h->fam_B.as<uint64_t>();
    v.fam_q = h->fam_q.as<uint8_t>();
    v.fam_u = h->fam_u.as<double>();
    v.fam_V = h->fam_V.as<double>();
    v.fam_v = h->fam_v.as<double>();
    v.ginfo = h->ginfo.as<uint4>();
    v.trec = h->trec.as<uint64_t>();
    v.famrec = h->famrec.as<uint64_t>();
    ck(cudaDeviceSynchronize(), "upload sync");
    *out = h.release();
  });
}

int qvmc_cuda_ham_create_from_index(qvmc_index_t idx, int device, qvmc_ham_t* out) {
  if (!idx) {
    g_error = "null index";
    return QVMC_ERR_INVALID_ARGUMENT;
  }
  const HostIndex& h = idx->idx;
  return qvmc_cuda_ham_create(h.n_qubits, h.n_words, h.n_xy(), h.xy.data(), h.offsets.data(), h.n_terms(),
                              h.coeff.data(), h.yz.data(), h.y_weight.data(), h.diag, device, out);
}

int qvmc_cuda_ham_destroy(qvmc_ham_t h) {
  return guarded([&] {
    if (!h) return;
    DeviceGuard dg(h->device);
    if (h->own) {
      cudaStreamSynchronize(h->own);
      cudaStreamDestroy(h->own);
    }
    for (auto& e : h->ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : h->ev_p)
      if (e) cudaEventDestroy(e);
    for (auto& e : h->ev_b) cudaEventDestroy(e);
    for (auto& e : h->ev_f)
      if (e) cudaEventDestroy(e);
    if (h->side) {
      cudaStreamSynchronize(h->side);
      cudaStreamDestroy(h->side);
    }
    if (h->log_host) cudaFreeHost(h->log_host);
    delete h;
  });
}

int qvmc_cuda_set_stream(qvmc_ham_t h, void* stream) {
  return guarded([&] {
    check_handle(h);
    h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own;
  });
}

int qvmc_cuda_set_speculative(qvmc_ham_t h, int on) {
  return guarded([&] {
    check_handle(h);
    DeviceGuard dg(h->device);
    if (!on && h->pending) resolve_pending(h);
    h->no_spec = on == 0;
  });
}

int qvmc_cuda_synchronize(qvmc_ham_t h) {
  return guarded([&] {
    check_handle(h);
    DeviceGuard dg(h->device);
    if (h->pending) resolve_pending(h);
    finish(h);
  });
}

int qvmc_cuda_last_stats(qvmc_ham_t h, qvmc_stats* out) {
  return guarded([&] {
    check_handle(h);
    if (!out) fail(QVMC_ERR_INVALID_ARGUMENT, "null stats");
    DeviceGuard dg(h->device);
    unsigned long long st[2];
    ck(cudaMemcpyAsync(st, static_cast<int*>(h->ctl.p) + 6, sizeof(st), cudaMemcpyDeviceToHost, h->stream), "stats");
    int mm[2];
    ck(cudaMemcpyAsync(mm, static_cast<int*>(h->ctl.p) + 2, sizeof(mm), cudaMemcpyDeviceToHost, h->stream), "mm");
    ck(cudaStreamSynchronize(h->stream), "sync");
    *out = h->last;
    if (h->timed) {
      ck(cudaEventElapsedTime(&out->table_ms, h->ev[0], h->ev[1]), "elapsed");
      ck(cudaEventElapsedTime(&out->rows_ms, h->ev[1], h->ev[2]), "elapsed");
      ck(cudaEventElapsedTime(&out->moments_ms, h->ev[2], h->ev[3]), "elapsed");
    }
    if (h->timed_f) {  // fused: one kernel does both; reported as search_ms
      ck(cudaEventElapsedTime(&out->search_ms, h->ev_f[0], h->ev_f[1]), "elapsed");
      out->eval_ms = 0.f;
    } else if (h->timed_b > 0) {  // pipelined: per-launch kernel times summed over the row batches
      out->search_ms = out->eval_ms = 0.f;
      for (int64_t b = 0; b < h->timed_b; ++b) {
        float ts = 0.f, te = 0.f;
        ck(cudaEventElapsedTime(&ts, h->ev_b[4 * b], h->ev_b[4 * b + 1]), "elapsed");
        ck(cudaEventElapsedTime(&te, h->ev_b[4 * b + 2], h->ev_b[4 * b + 3]), "elapsed");
        out->search_ms += ts;
        out->eval_ms += te;
      }
    }
    out->candidates = st[0];
    out->pairs = st[1];
  });
}

int qvmc_cuda_pairs(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, int mem, int backend, int auto_threshold,
                    uint64_t* n_pairs, uint64_t* ops, int* backend_used) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (n_unq < 0 || n_unq >= 0xFFFFFFFFll) fail(QVMC_ERR_INVALID_ARGUMENT, "n_unq out of range");
    if (n_unq > 0 && !keys) fail(QVMC_ERR_INVALID_ARGUMENT, "null keys");
    if (backend < QVMC_BACKEND_TERMS || backend > QVMC_BACKEND_AUTO)
      fail(QVMC_ERR_INVALID_ARGUMENT, "unknown coupling backend");
    DeviceGuard dg(h->device);
    int used = backend;
    if (backend == QVMC_BACKEND_AUTO)  // coupling.cpp:157-161
      used = n_unq < auto_threshold ? QVMC_BACKEND_BATCH : QVMC_BACKEND_TRIE;
    const int W = h->W;
    const uint64_t* dkeys = stage(h, h->keys, keys, static_cast<size_t>(n_unq) * W, mem);
    record_stats(h, n_unq);
    h->pairs_rows = n_unq;
    h->n_pairs = 0;
    ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 6, 0, 4 * sizeof(int), h->stream), "memset stats");
    uint64_t total = 0;
    if (n_unq > 0) {
      ck(cudaEventRecord(h->ev[0], h->stream), "event");
      DISPATCH_W(W, launch_table_build<WW>(h, dkeys, n_unq));
      {
        const int err = read_err_and_reset(h);
        if (err) raise_device_err(err);
      }
      const RowPlan P = plan_rows(h, n_unq);
      note_plan(h, P);
      if (P.join) DISPATCH_W(W, build_join_index<WW>(h, dkeys, n_unq, P));
      ck(cudaEventRecord(h->ev[1], h->stream), "event");
      h->counts.ensure((n_unq + 1) * sizeof(uint32_t));
      h->row_off.ensure((n_unq + 1) * sizeof(uint64_t));
      RowOut O{};
      O.counts = h->counts.as<uint32_t>();
      DISPATCH_W(W, (run_rows<WW, kModeCount>(h, dkeys, 0, n_unq, P, O)));
      ck(cudaEventRecord(h->ev[2], h->stream), "event");  // stats: rows_ms = the counting pass
      // exclusive scan of the per-row counts (as u64)
      ck(cudaMemsetAsync(h->counts.as<uint32_t>() + n_unq, 0, sizeof(uint32_t), h->stream), "memset");
      size_t tmp = 0;
      uint64_t* roff = h->row_off.as<uint64_t>();
      auto in_it = h->counts.as<uint32_t>();
      ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in_it, roff, n_unq + 1, h->stream), "scan size");
      h->cub_tmp.ensure(tmp + 16);
      ck(cub::DeviceScan::ExclusiveSum(h->cub_tmp.p, tmp, in_it, roff, n_unq + 1, h->stream), "scan");
      ++g_launches;
      ck(cudaMemcpyAsync(&total, roff + n_unq, sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream), "D2H total");
      ck(cudaStreamSynchronize(h->stream), "sync");
      if (total >= (1ull << 31)) fail(QVMC_ERR_RUNTIME, "coupled-pair list exceeds 2^31 entries");
      h->xp_a.ensure(total * 4 + 16);
      h->g_a.ensure(total * 4 + 16);
      h->xp_b.ensure(total * 4 + 16);
      h->g_b.ensure(total * 4 + 16);
      O = RowOut{};
      O.row_off = roff;
      O.xp_out = h->xp_a.as<uint32_t>();
      O.g_out = h->g_a.as<uint32_t>();
      DISPATCH_W(W, (run_rows<WW, kModeEmit>(h, dkeys, 0, n_unq, P, O)));
      // canonical order inside each row: by x' (coupling.cpp:49-52)
      tmp = 0;
      ck(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tmp, h->xp_a.as<uint32_t>(), h->xp_b.as<uint32_t>(),
                                                   h->g_a.as<uint32_t>(), h->g_b.as<uint32_t>(),
                                                   static_cast<int>(total), static_cast<int>(n_unq), roff, roff + 1,
                                                   h->stream),
         "segsort size");
      h->cub_tmp.ensure(tmp + 16);
      ck(cub::DeviceSegmentedSort::StableSortPairs(h->cub_tmp.p, tmp, h->xp_a.as<uint32_t>(), h->xp_b.as<uint32_t>(),
                                                   h->g_a.as<uint32_t>(), h->g_b.as<uint32_t>(),
                                                   static_cast<int>(total), static_cast<int>(n_unq), roff, roff + 1,
                                                   h->stream),
         "segsort");
      ++g_launches;
      ck(cudaEventRecord(h->ev[3], h->stream), "event");
      h->timed = true;
      const int err = read_err_and_reset(h);
      if (err) raise_device_err(err);
    }
    h->n_pairs = total;
    unsigned long long st[2] = {0, 0};
    ck(cudaMemcpy(st, static_cast<int*>(h->ctl.p) + 6, sizeof(st), cudaMemcpyDeviceToHost), "stats");
    const uint64_t probed = st[0] + (h->diag >= 0 ? static_cast<uint64_t>(n_unq) : 0);
    const uint64_t n64 = static_cast<uint64_t>(n_unq);
    if (n_pairs) *n_pairs = total;
    if (ops)
      *ops = used == QVMC_BACKEND_TERMS ? n64 * h->n_xy : used == QVMC_BACKEND_BATCH ? n64 * n64 : probed;
    if (backend_used) *backend_used = used;
  });
}

namespace {
__global__ void k_pack_entries(const uint64_t* __restrict__ row_off, int64_t n, const uint32_t* __restrict__ xp,
                               const uint32_t* __restrict__ g, uint32_t* out3) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (uint64_t e = row_off[i]; e < row_off[i + 1]; ++e) {
      out3[3 * e] = static_cast<uint32_t>(i);
      out3[3 * e + 1] = xp[e];
      out3[3 * e + 2] = g[e];
    }
}
}  // namespace

int qvmc_cuda_pairs_fetch(qvmc_ham_t h, uint32_t* out_entries, int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (h->n_pairs == 0) return;
    if (!out_entries) fail(QVMC_ERR_INVALID_ARGUMENT, "null output");
    DeviceGuard dg(h->device);
    uint32_t* dst = out_entries;
    if (mem == QVMC_MEM_HOST) {
      h->entries.ensure(h->n_pairs * 12);
      dst = h->entries.as<uint32_t>();
    }
    const int grid = static_cast<int>(std::min<int64_t>((h->pairs_rows + kThreads - 1) / kThreads, grid_for(h, 8)));
    k_pack_entries<<<std::max(grid, 1), kThreads, 0, h->stream>>>(h->row_off.as<uint64_t>(), h->pairs_rows,
                                                                  h->xp_b.as<uint32_t>(), h->g_b.as<uint32_t>(), dst);
    ck_launch("pack entries");
    if (mem == QVMC_MEM_HOST)
      ck(cudaMemcpyAsync(out_entries, dst, h->n_pairs * 12, cudaMemcpyDeviceToHost, h->stream), "D2H entries");
    ck(cudaStreamSynchronize(h->stream), "sync");
  });
}

int qvmc_cuda_pair_elements(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, uint64_t n_pairs,
                            const uint32_t* entries, double* out_h, uint8_t* out_class, int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (n_unq < 0 || (n_unq > 0 && !keys) || (n_pairs > 0 && (!entries || !out_h)))
      fail(QVMC_ERR_INVALID_ARGUMENT, "null or negative argument");
    if (n_pairs == 0) return;
    DeviceGuard dg(h->device);
    const int W = h->W;
    const uint64_t* dkeys = stage(h, h->keys, keys, static_cast<size_t>(n_unq) * W, mem);
    const uint32_t* de = stage(h, h->in_entries, entries, n_pairs * 3, mem);
    double2* dh = reinterpret_cast<double2*>(out_h);
    uint8_t* dc = out_class;
    if (mem == QVMC_MEM_HOST) {
      h->out_h.ensure(n_pairs * 16);
      dh = h->out_h.as<double2>();
      dc = nullptr;
      if (out_class) {
        h->out_class.ensure(n_pairs + 16);
        dc = h->out_class.as<uint8_t>();
      }
    }
    const int grid = static_cast<int>(std::min<uint64_t>((n_pairs + kThreads - 1) / kThreads, grid_for(h, 8)));
    DISPATCH_W(W, (k_pair_elements<WW><<<grid, kThreads, 0, h->stream>>>(h->view, dkeys, n_unq, de, n_pairs, dh, dc,
                                                                       static_cast<int*>(h->ctl.p))));
    ck_launch("pair elements");
    if (mem == QVMC_MEM_HOST) {
      ck(cudaMemcpyAsync(out_h, dh, n_pairs * 16, cudaMemcpyDeviceToHost, h->stream), "D2H h");
      if (out_class) ck(cudaMemcpyAsync(out_class, dc, n_pairs, cudaMemcpyDeviceToHost, h->stream), "D2H class");
    }
    finish(h);
  });
}

int qvmc_cuda_pair_elements_fused(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, uint64_t n_pairs,
                                  const uint32_t* entries, double* out_h, uint8_t* out_kind, int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (n_unq < 0 || (n_unq > 0 && !keys) || (n_pairs > 0 && (!entries || !out_h || !out_kind)))
      fail(QVMC_ERR_INVALID_ARGUMENT, "null or negative argument");
    if (n_pairs == 0 || n_unq == 0) return;
    DeviceGuard dg(h->device);
    const int W = h->W;
    const uint64_t* dkeys = stage(h, h->keys, keys, static_cast<size_t>(n_unq) * W, mem);
    const uint32_t* de = stage(h, h->in_entries, entries, n_pairs * 3, mem);
    double2* dh = reinterpret_cast<double2*>(out_h);
    uint8_t* dk = out_kind;
    if (mem == QVMC_MEM_HOST) {
      h->out_h.ensure(n_pairs * 16);
      h->out_class.ensure(n_pairs + 16);
      dh = h->out_h.as<double2>();
      dk = h->out_class.as<uint8_t>();
    }
    int* err = static_cast<int*>(h->ctl.p);
    h->p_rlo.ensure(n_unq * 4 + 16);
    h->p_rhi.ensure(n_unq * 4 + 16);
    ck(cudaMemsetAsync(h->p_rlo.p, 0, n_unq * 4, h->stream), "memset rows");
    ck(cudaMemsetAsync(h->p_rhi.p, 0, n_unq * 4, h->stream), "memset rows");
    const int g1 = static_cast<int>(std::min<uint64_t>((n_pairs + kThreads - 1) / kThreads, grid_for(h, 8)));
    k_check_sorted<<<g1, kThreads, 0, h->stream>>>(de, n_pairs, n_unq, err);
    ck_launch("check pairs");
    k_pair_rows<<<g1, kThreads, 0, h->stream>>>(de, n_pairs, n_unq, h->p_rlo.as<uint32_t>(), h->p_rhi.as<uint32_t>());
    ck_launch("pair rows");
    const int grid = static_cast<int>(std::min<int64_t>((n_unq + kWarps - 1) / kWarps, grid_for(h, 8)));
    RowPlan P0{};
    DISPATCH_W(W, (k_pair_records<WW><<<grid, kThreads, 0, h->stream>>>(
                      h->view, join_view(h, P0), h->gkey.as<uint32_t>(), dkeys, n_unq, de, h->p_rlo.as<uint32_t>(),
                      h->p_rhi.as<uint32_t>(), dh, dk, err)));
    ck_launch("pair records");
    if (mem == QVMC_MEM_HOST) {
      ck(cudaMemcpyAsync(out_h, dh, n_pairs * 16, cudaMemcpyDeviceToHost, h->stream), "D2H h");
      ck(cudaMemcpyAsync(out_kind, dk, n_pairs, cudaMemcpyDeviceToHost, h->stream), "D2H kind");
    }
    finish(h);
  });
}

int qvmc_cuda_local_energies(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                             const double* phase, uint64_t n_pairs, const uint32_t* entries, double* out_eloc,
                             int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (n_unq < 0 || (n_unq > 0 && (!keys || !log_amp || !phase || !out_eloc)) || (n_pairs > 0 && !entries))
      fail(QVMC_ERR_INVALID_ARGUMENT, "null or negative argument");
    if (n_unq == 0) return;
    DeviceGuard dg(h->device);
    const int W = h->W;
    const uint64_t* dkeys = stage(h, h->keys, keys, static_cast<size_t>(n_unq) * W, mem);
    const double* dla = stage(h, h->la, log_amp, n_unq, mem);
    const double* dph = stage(h, h->ph, phase, n_unq, mem);
    const uint32_t* de = stage(h, h->in_entries, entries, n_pairs * 3, mem);
    double2* dout = reinterpret_cast<double2*>(out_eloc);
    if (mem == QVMC_MEM_HOST) {
      h->eloc.ensure(n_unq * 16);
      dout = h->eloc.as<double2>();
    }
    int* err = static_cast<int*>(h->ctl.p);
    h->p_rlo.ensure(n_unq * 4 + 16);
    h->p_rhi.ensure(n_unq * 4 + 16);
    ck(cudaMemsetAsync(h->p_rlo.p, 0, n_unq * 4, h->stream), "memset rows");
    ck(cudaMemsetAsync(h->p_rhi.p, 0, n_unq * 4, h->stream), "memset rows");
    if (n_pairs > 0) {
      const int g1 = static_cast<int>(std::min<uint64_t>((n_pairs + kThreads - 1) / kThreads, grid_for(h, 8)));
      k_check_sorted<<<g1, kThreads, 0, h->stream>>>(de, n_pairs, n_unq, err);
      ck_launch("check pairs");
      k_pair_rows<<<g1, kThreads, 0, h->stream>>>(de, n_pairs, n_unq, h->p_rlo.as<uint32_t>(), h->p_rhi.as<uint32_t>());
      ck_launch("pair rows");
    }
    h->cs.ensure(n_unq * 16 + 16);
    {
      const int grid = static_cast<int>(std::min<int64_t>((n_unq + kThreads - 1) / kThreads, grid_for(h, 8)));
      k_cos_sin<<<std::max(grid, 1), kThreads, 0, h->stream>>>(dph, n_unq, h->cs.as<double2>());
      ck_launch("cos sin");
    }
    const int grid = static_cast<int>(std::min<int64_t>((n_unq + kWarps - 1) / kWarps, grid_for(h, 8)));
    RowPlan P0{};
    DISPATCH_W(W, (k_pairs_eloc2<WW><<<grid, kThreads, 0, h->stream>>>(
                      h->view, join_view(h, P0), h->gkey.as<uint32_t>(), dkeys, dla, h->cs.as<double2>(), n_unq, de,
                      h->p_rlo.as<uint32_t>(), h->p_rhi.as<uint32_t>(), dout, err)));
    ck_launch("local energies");
    if (mem == QVMC_MEM_HOST) {
      ck(cudaMemcpyAsync(out_eloc, dout, n_unq * 16, cudaMemcpyDeviceToHost, h->stream), "D2H eloc");
      finish(h);
    }
  });
}

int qvmc_cuda_energy_moments(qvmc_ham_t h, int64_t n, const double* log_prob, double log_norm, const double* eloc,
                             double* out_moments, double* out_weights, int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (n < 0 || (n > 0 && (!log_prob || !eloc)) || !out_moments) fail(QVMC_ERR_INVALID_ARGUMENT, "null argument");
    DeviceGuard dg(h->device);
    const double* dlp = stage(h, h->lp, log_prob, n, mem);
    const double2* de = reinterpret_cast<const double2*>(stage(h, h->eloc, eloc, 2 * n, mem));
    double* dm = out_moments;
    double* dw = out_weights;
    if (mem == QVMC_MEM_HOST) {
      h->moments.ensure(8 * sizeof(double));
      dm = h->moments.as<double>();
      dw = nullptr;
      if (out_weights) {
        h->weights.ensure(n * 8 + 16);
        dw = h->weights.as<double>();
      }
    }
    compute_moments(h, dlp, log_norm, de, n, dm, dw);
    if (mem == QVMC_MEM_HOST) {
      ck(cudaMemcpyAsync(out_moments, dm, 5 * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "D2H moments");
      if (out_weights && n)
        ck(cudaMemcpyAsync(out_weights, dw, n * 8, cudaMemcpyDeviceToHost, h->stream), "D2H weights");
      finish(h);
    }
  });
}

int qvmc_cuda_eloc_fused(qvmc_ham_t h, int64_t n_unq, const uint64_t* keys, const double* log_amp,
                         const double* phase, const double* log_prob, double log_norm, int64_t row_begin,
                         int64_t row_end, double* out_eloc, double* out_moments, int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (n_unq < 0 || n_unq >= 0xFFFFFFFFll) fail(QVMC_ERR_INVALID_ARGUMENT, "n_unq out of range");
    if (row_begin < 0 || row_end < row_begin || row_end > n_unq) fail(QVMC_ERR_INVALID_ARGUMENT, "bad row range");
    if (n_unq > 0 && (!keys || !log_amp || !phase)) fail(QVMC_ERR_INVALID_ARGUMENT, "null sample arrays");
    if (out_moments && row_end > row_begin && !log_prob) fail(QVMC_ERR_INVALID_ARGUMENT, "moments need log_prob");
    DeviceGuard dg(h->device);
    if (h->pending) resolve_pending(h);  // an earlier speculative call is checked first
    // speculative: device memory and a cached sector plan for this sample-set size -> no host
    // synchronisation anywhere in the call (CUDA-graph capturable once the buffers are sized)
    const bool spec = mem == QVMC_MEM_DEVICE && !h->no_spec && h->plan_ok && h->plan_n == n_unq && n_unq > 0 &&
                      h->walk_world <= 1;
    const int W = h->W;
    const int64_t rows = row_end - row_begin;
    const uint64_t* dkeys = stage(h, h->keys, keys, static_cast<size_t>(n_unq) * W, mem);
    // host amplitudes: copied on a second stream while the sample-set index is built from the keys
    cudaStream_t main_stream = h->stream;
    if (mem == QVMC_MEM_HOST && n_unq > 0) {
      if (!h->side) {
        ck(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking), "stream create");
        for (auto& e : h->ev_p) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
      }
      ck(cudaEventRecord(h->ev_p[6], main_stream), "event");  // after earlier work on the buffers
      ck(cudaStreamWaitEvent(h->side, h->ev_p[6], 0), "wait");
      h->stream = h->side;
    }
    const double* dla = stage(h, h->la, log_amp, n_unq, mem);
    const double* dph = stage(h, h->ph, phase, n_unq, mem);
    const double* dlp = log_prob ? stage(h, h->lp, log_prob, n_unq, mem) : nullptr;
    const bool h2d_async = h->stream != main_stream;
    if (h2d_async) {
      ck(cudaEventRecord(h->ev_p[7], h->side), "event");
      h->stream = main_stream;
    }
    auto wait_amplitudes = [&] {
      if (h2d_async) ck(cudaStreamWaitEvent(h->stream, h->ev_p[7], 0), "wait");
    };
    double2* deloc = reinterpret_cast<double2*>(out_eloc);
    if (mem == QVMC_MEM_HOST || !out_eloc) {
      h->eloc.ensure(std::max<int64_t>(rows, 1) * 16);
      deloc = h->eloc.as<double2>();
    }
    record_stats(h, rows);
    ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 6, 0, 4 * sizeof(int), h->stream), "memset stats");
    ck(cudaEventRecord(h->ev[0], h->stream), "event");
    RowPlan P;
    bool fused_ok = false;  // QVMC_FUSED=1 and a minority set the fused rings carry
    RowSet R{};
    const uint64_t* rkeys = dkeys;
    const double2* rcs = nullptr;
    if (n_unq > 0) {
      // sector test first: the join path (row search, modes 0/1) needs no sample
      // hash table (duplicate keys are caught by the search), other paths build it
      ck(cudaMemsetAsync(static_cast<int*>(h->ctl.p) + 2, 0, 2 * sizeof(int), h->stream), "memset popcount range");
      const int pgrid = static_cast<int>(std::min<int64_t>((n_unq + kThreads - 1) / kThreads, grid_for(h, 4)));
      DISPATCH_W(W, (k_popc_range<WW><<<std::max(pgrid, 1), kThreads, 0, h->stream>>>(dkeys, n_unq,
                                                                                      static_cast<int*>(h->ctl.p) + 2)));
      ck_launch("popcount range");
      if (spec) {
        P = cached_plan(h);
        k_plan_check<<<1, 1, 0, h->stream>>>(static_cast<int*>(h->ctl.p) + 2, h->plan_mm[0], h->plan_mm[1],
                                             static_cast<int*>(h->ctl.p));
        ck_launch("plan check");
      } else {
        P = plan_rows(h, n_unq);
      }
      note_plan(h, P);
      fused_ok = h->fused && P.s <= kFusedMaxMinority;
      if (!P.join) DISPATCH_W(W, launch_table_build<WW>(h, dkeys, n_unq));
      if (P.join) {
        DISPATCH_W(W, R = sort_for_locality<WW>(h, rkeys, n_unq, row_begin, row_end, P));
        if (h->view.n_res) DISPATCH_W(W, launch_table_build<WW>(h, rkeys, n_unq));  // residual probes: sorted ids
        // symmetric when every row of the set is evaluated by this call, or by the ranks of a sharded call
        const bool sym = h->sym && !h->sym_off_once && !fused_ok && (R.list == nullptr || h->shard_sym);
        h->sym_off_once = false;
        h->shard_sym_active = sym && h->shard_sym;
        DISPATCH_W(W, build_join_index<WW>(h, rkeys, n_unq, P, sym));
        wait_amplitudes();  // a host caller's amplitude upload ran beside the index build
        gather_records(h, dla, dph, n_unq);
      } else {
        wait_amplitudes();
        h->cs.ensure(n_unq * 16 + 16);
        const int grid = static_cast<int>(std::min<int64_t>((n_unq + kThreads - 1) / kThreads, grid_for(h, 8)));
        k_cos_sin<<<std::max(grid, 1), kThreads, 0, h->stream>>>(dph, n_unq, h->cs.as<double2>());
        ck_launch("cos sin");
        rcs = h->cs.as<double2>();
      }
    }
    ck(cudaEventRecord(h->ev[1], h->stream), "event");
    if (n_unq > 0) {
      RowOut O{};
      O.eloc = deloc;
      O.la = dla;
      O.ph = dph;
      O.cs = rcs;
      h->last_rows = R;
      if (P.join && fused_ok) {
        DISPATCH_W(W, (run_join_fused<WW>(h, rkeys, R, P, deloc)));
      } else if (P.join) {
        bool redo = false;
        DISPATCH_W(W, (redo = run_join_pipelined<WW>(h, rkeys, n_unq, R, P, deloc, spec)));
        if (redo && (h->shard_sym || h->dist_comm)) {  // sharded: every rank must take the same path
          h->fix_range_flag = true;                   // (reported through the moment exchange)
          redo = false;
        }
        if (redo) {  // exchange symmetry left the fixed-point range: rebuild unpaired and rerun
          h->shard_sym_active = false;
          DISPATCH_W(W, build_join_index<WW>(h, rkeys, n_unq, P, false));
          DISPATCH_W(W, (run_join_pipelined<WW>(h, rkeys, n_unq, R, P, deloc, false)));
        }
      } else {
        int64_t b = row_begin, e = row_end;
        RowOut Os = O;
        if (h->walk_world > 1) {  // sharded, strided mode: rows without the join are split contiguously
          shard_range(n_unq, h->walk_world, h->walk_rank, b, e);
          Os.eloc = deloc + (b - row_begin);
        }
        DISPATCH_W(W, (launch_rows<WW, kModeEloc>(h, dkeys, b, e, Os)));
      }
    }
    ck(cudaEventRecord(h->ev[2], h->stream), "event");
    double* dm = out_moments;
    if (out_moments) {
      if (mem == QVMC_MEM_HOST) {
        h->moments.ensure(8 * sizeof(double));
        dm = h->moments.as<double>();
      }
      compute_moments(h, dlp ? dlp + row_begin : nullptr, log_norm, deloc, rows, dm, nullptr);
    }
    ck(cudaEventRecord(h->ev[3], h->stream), "event");
    h->timed = true;
    if (!P.join) h->shard_sym_active = false;
    if (spec) {
      h->pending = true;
      h->pend = {n_unq, row_begin, row_end, keys, log_amp, phase, log_prob, log_norm, out_eloc, out_moments};
      h->pend_stream = h->stream;
    }
    if (mem == QVMC_MEM_HOST) {
      if (out_eloc && rows)
        ck(cudaMemcpyAsync(out_eloc, deloc, rows * 16, cudaMemcpyDeviceToHost, h->stream), "D2H eloc");
      if (out_moments) ck(cudaMemcpyAsync(out_moments, dm, 5 * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "D2H");
      finish(h);
    }
  });
}

// ------------------------------------------------------------------ sharded path

int qvmc_shard_bounds(int64_t n_total, int world, int rank, int64_t* begin, int64_t* end) {
  return guarded([&] {
    if (n_total < 0 || world < 1 || rank < 0 || rank >= world) fail(QVMC_ERR_INVALID_ARGUMENT, "bad shard request");
    int64_t b, e;
    shard_range(n_total, world, rank, b, e);
    if (begin) *begin = b;
    if (end) *end = e;
  });
}

int qvmc_cuda_comm_unique_id(void* out, uint64_t out_bytes) {
  return guarded([&] {
    if (!out || out_bytes < sizeof(ncclUniqueId)) fail(QVMC_ERR_INVALID_ARGUMENT, "unique id buffer < 128 bytes");
    ncclUniqueId id;
    nccl_ck(nccl_or_fail().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  });
}

int qvmc_cuda_comm_init_nccl(int device, int world, int rank, const void* unique_id, qvmc_comm_t* out) {
  return guarded([&] {
    if (!out || !unique_id) fail(QVMC_ERR_INVALID_ARGUMENT, "null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(QVMC_ERR_INVALID_ARGUMENT, "bad world/rank");
    const NcclApi& a = nccl_or_fail();
    DeviceGuard dg(device);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    auto c = std::make_unique<qvmc_comm_s>();
    c->world = world;
    c->rank = rank;
    nccl_ck(a.CommInitRank(&c->nccl, world, id, rank), "ncclCommInitRank");
    c->owns = true;
    *out = c.release();
  });
}

int qvmc_cuda_comm_wrap_nccl(void* nccl_comm, int world, int rank, qvmc_comm_t* out) {
  return guarded([&] {
    if (!out || !nccl_comm) fail(QVMC_ERR_INVALID_ARGUMENT, "null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(QVMC_ERR_INVALID_ARGUMENT, "bad world/rank");
    nccl_or_fail();
    auto c = std::make_unique<qvmc_comm_s>();
    c->world = world;
    c->rank = rank;
    c->nccl = static_cast<ncclComm_t>(nccl_comm);
    *out = c.release();
  });
}

int qvmc_cuda_comm_init_host(int world, int rank, qvmc_host_allgather_fn all_gather, void* ctx, qvmc_comm_t* out) {
  return guarded([&] {
    if (!out || !all_gather) fail(QVMC_ERR_INVALID_ARGUMENT, "null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(QVMC_ERR_INVALID_ARGUMENT, "bad world/rank");
    auto c = std::make_unique<qvmc_comm_s>();
    c->world = world;
    c->rank = rank;
    c->host_ag = all_gather;
    c->ctx = ctx;
    *out = c.release();
  });
}

int qvmc_cuda_comm_destroy(qvmc_comm_t c) {
  return guarded([&] {
    if (!c) return;
    std::unique_ptr<qvmc_comm_s> own(c);
    if (c->hsend) cudaFreeHost(c->hsend);
    if (c->hrecv) cudaFreeHost(c->hrecv);
    if (c->owns && c->nccl) nccl_ck(nccl_api().CommDestroy(c->nccl), "ncclCommDestroy");
  });
}

int qvmc_cuda_eloc_sharded(qvmc_ham_t h, qvmc_comm_t comm, int64_t n_total, const uint64_t* keys,
                           const double* log_amp, const double* phase, const double* log_prob, double log_norm,
                           double* out_eloc, double* out_moments, int mem) {
  return guarded([&] {
    check_handle(h);
    check_mem(mem);
    if (!comm) fail(QVMC_ERR_INVALID_ARGUMENT, "null communicator");
    if (n_total < 0 || n_total >= 0xFFFFFFFFll) fail(QVMC_ERR_INVALID_ARGUMENT, "n_unq out of range");
    const int world = comm->world, rank = comm->rank;
    int64_t r0, r1;
    shard_range(n_total, world, rank, r0, r1);
    const int64_t rows = r1 - r0;
    const int64_t max_rows = (n_total + world - 1) / world;
    if (rows > 0 && (!keys || !log_amp || !phase)) fail(QVMC_ERR_INVALID_ARGUMENT, "null sample arrays");
    if (out_moments && n_total > 0 && !log_prob) fail(QVMC_ERR_INVALID_ARGUMENT, "moments need log_prob");
    DeviceGuard dg(h->device);
    const int W = h->W;
    const uint64_t* dk = stage(h, h->s_keys, keys, static_cast<size_t>(rows) * W, mem);
    const double* dla = stage(h, h->s_la, log_amp, rows, mem);
    const double* dph = stage(h, h->s_ph, phase, rows, mem);
    const double* dlp = log_prob ? stage(h, h->s_lp, log_prob, rows, mem) : nullptr;
    const size_t rec = static_cast<size_t>(W + 3) * 8;
    const size_t block = std::max<size_t>(static_cast<size_t>(max_rows) * rec, 8);
    h->g_send.ensure(block + 16);
    h->g_recv.ensure(block * world + 16);
    const int pgrid = static_cast<int>(std::min<int64_t>((std::max<int64_t>(rows, 1) + kThreads - 1) / kThreads,
                                                         grid_for(h, 8)));
    if (rows > 0) {
      DISPATCH_W(W, (k_pack_shard<WW><<<pgrid, kThreads, 0, h->stream>>>(dk, dla, dph, dlp, rows,
                                                                         h->g_send.as<uint64_t>())));
      ck_launch("pack shard");
    }
    comm_all_gather(comm, h->g_send.p, h->g_recv.p, block, h->stream);
    h->g_keys.ensure(static_cast<size_t>(n_total) * W * 8 + 16);
    h->g_la.ensure(static_cast<size_t>(n_total) * 8 + 16);
    h->g_ph.ensure(static_cast<size_t>(n_total) * 8 + 16);
    h->g_lp.ensure(static_cast<size_t>(n_total) * 8 + 16);
    if (n_total > 0) {
      const int ugrid = static_cast<int>(std::min<int64_t>((n_total + kThreads - 1) / kThreads, grid_for(h, 8)));
      DISPATCH_W(W, (k_unpack_shards<WW><<<ugrid, kThreads, 0, h->stream>>>(
                        h->g_recv.as<uint64_t>(), world, max_rows, n_total, h->g_keys.as<uint64_t>(),
                        h->g_la.as<double>(), h->g_ph.as<double>(), h->g_lp.as<double>())));
      ck_launch("unpack shards");
    }
    // E_loc of this rank's rows against the gathered set + its moments. Symmetric across ranks:
    // each rank walks its rows' partners after them, the mirrored fixed-point sums of all ranks are
    // added (exact integer all-reduce), so every row gets exactly the single-GPU symmetric result
    double* deloc = (mem == QVMC_MEM_DEVICE) ? out_eloc : nullptr;
    h->g_mom.ensure(8 * sizeof(double));
    ck(cudaMemsetAsync(h->g_mom.p, 0, 8 * sizeof(double), h->stream), "memset moments");
    h->shard_sym = world > 1;
    h->fix_range_flag = false;
    h->dist_comm = (world > 1 && h->dist_index) ? comm : nullptr;
    // strided walk (default for world > 1): this rank walks sorted positions rank, rank + world, ...
    // into a zeroed n_total-row vector in caller order; each row is written by exactly one rank, so an
    // integer all-reduce of the bit patterns assembles the single-GPU result exactly on every rank
    const bool strided = world > 1 && h->strided_shards && n_total > 0;
    if (strided) {
      h->eloc.ensure(static_cast<size_t>(n_total) * 16);
      ck(cudaMemsetAsync(h->eloc.p, 0, static_cast<size_t>(n_total) * 16, h->stream), "memset rows");
      h->walk_world = world;
      h->walk_rank = rank;
    }
    const int st = strided ? qvmc_cuda_eloc_fused(h, n_total, h->g_keys.as<uint64_t>(), h->g_la.as<double>(),
                                                  h->g_ph.as<double>(), nullptr, log_norm, 0, n_total, nullptr,
                                                  nullptr, QVMC_MEM_DEVICE)
                           : qvmc_cuda_eloc_fused(h, n_total, h->g_keys.as<uint64_t>(), h->g_la.as<double>(),
                                                  h->g_ph.as<double>(), log_prob ? h->g_lp.as<double>() : nullptr,
                                                  log_norm, r0, r1, deloc,
                                                  out_moments ? h->g_mom.as<double>() : nullptr, QVMC_MEM_DEVICE);
    h->shard_sym = false;
    h->dist_comm = nullptr;
    h->walk_world = 0;
    if (st != QVMC_OK) fail(st, g_error);
    if (strided) {
      double2* de = h->eloc.as<double2>();
      if (h->shard_sym_active) {
        h->shard_sym_active = false;
        comm_all_reduce_u64(comm, h->s_fix.as<unsigned long long>(), static_cast<size_t>(n_total) * 4, h->stream,
                            h->g_recv);
        const RowSet R = h->last_rows;
        const int fg = static_cast<int>(std::min<int64_t>((R.n_rows + kThreads - 1) / kThreads, grid_for(h, 8)));
        k_add_fix<<<std::max(fg, 1), kThreads, 0, h->stream>>>(R, h->s_fix.as<unsigned long long>(), de);
        ck_launch("add mirrored sums");
      }
      comm_all_reduce_u64(comm, h->eloc.as<unsigned long long>(), static_cast<size_t>(n_total) * 2, h->stream,
                          h->g_recv);
      if (out_moments && rows > 0)
        compute_moments(h, log_prob ? h->g_lp.as<double>() + r0 : nullptr, log_norm, de + r0, rows,
                        h->g_mom.as<double>(), nullptr);
      if (mem == QVMC_MEM_DEVICE && out_eloc && rows > 0)
        ck(cudaMemcpyAsync(out_eloc, de + r0, rows * 16, cudaMemcpyDeviceToDevice, h->stream), "copy rows");
    } else if (h->shard_sym_active) {
      h->shard_sym_active = false;
      comm_all_reduce_u64(comm, h->s_fix.as<unsigned long long>(), static_cast<size_t>(n_total) * 4, h->stream,
                          h->g_recv);
      double2* de = deloc ? reinterpret_cast<double2*>(deloc) : h->eloc.as<double2>();
      const RowSet R = h->last_rows;
      const int fg = static_cast<int>(std::min<int64_t>((R.n_rows + kThreads - 1) / kThreads, grid_for(h, 8)));
      k_add_fix<<<std::max(fg, 1), kThreads, 0, h->stream>>>(R, h->s_fix.as<unsigned long long>(), de);
      ck_launch("add mirrored sums");
      if (out_moments)  // the moments of the finished rows (the fused call's were taken before the fix)
        compute_moments(h, log_prob ? h->g_lp.as<double>() + r0 : nullptr, log_norm, de, rows,
                        h->g_mom.as<double>(), nullptr);
    }
    const bool flagged = world > 1 && h->sym && !(h->fused && h->last.minority_count <= kFusedMaxMinority);  // symmetric: the range flag too
    if (flagged) {
      const double f = h->fix_range_flag ? 1.0 : 0.0;
      ck(cudaMemcpyAsync(h->g_mom.as<double>() + 7, &f, sizeof(double), cudaMemcpyHostToDevice, h->stream), "flag");
    }
    if (out_moments || flagged) {  // per-rank moments gathered, summed in rank order
      h->g_moms.ensure(static_cast<size_t>(world) * 8 * sizeof(double) + 16);
      comm_all_gather(comm, h->g_mom.p, h->g_moms.p, 8 * sizeof(double), h->stream);
      if (flagged) {
        std::vector<double> all(static_cast<size_t>(world) * 8);
        ck(cudaMemcpyAsync(all.data(), h->g_moms.p, all.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream),
           "D2H flags");
        ck(cudaStreamSynchronize(h->stream), "sync");
        for (int r = 0; r < world; ++r)
          if (all[static_cast<size_t>(r) * 8 + 7] != 0.0)
            fail(QVMC_ERR_RUNTIME, "a mirrored local-energy contribution exceeded the exact fixed-point range "
                                   "(|value| >= 2^46): rerun with QVMC_SYMMETRIC=0");
      }
    }
    if (out_moments) {
      double* dm = out_moments;
      if (mem == QVMC_MEM_HOST) {
        h->moments.ensure(8 * sizeof(double));
        dm = h->moments.as<double>();
      }
      k_sum_rank_moments<<<1, 32, 0, h->stream>>>(h->g_moms.as<double>(), world, dm);
      ck_launch("rank moments");
      if (mem == QVMC_MEM_HOST)
        ck(cudaMemcpyAsync(out_moments, dm, 5 * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "D2H");
    }
    if (mem == QVMC_MEM_HOST) {
      if (out_eloc && rows)
        ck(cudaMemcpyAsync(out_eloc, h->eloc.as<double2>() + (strided ? r0 : 0), rows * 16, cudaMemcpyDeviceToHost,
                           h->stream), "D2H eloc");
      finish(h);
    }
  });
}

// ------------------------------------------------------------------ amplitude model
// AnqsModel (model.cpp) on the device: layout + sector checks as in the
// reference constructor (model.cpp:33-45, :47-97), parameters re-laid out per
// set_params (qvmc_model.cuh BlockLayout).
}  // extern "C"

struct qvmc_model_s {
  int device = 0;
  int n = 0, W = 0, bits = 6, n_e = 0, spin = 0, n_up = 0, hidden = 64, n_qudits = 0;
  int64_t n_params = 0;
  bool has_params = false;
  bool tiled = true;  // warp-tiled (qudit, head) CTAs (default); QVMC_MODEL_TILED=0: one CTA per sample tile
  int sms = 148;
  cudaStream_t own = nullptr, stream = nullptr;
  DBuf P, keys, la, ph, lp, part, out2, lse;
  // sampler (sample_without_replacement): two beams, the conditional table, candidates
  DBuf bk[2], blp[2], bpert[2], cond, c_key, c_key2, c_slot, c_slot2, c_bv, c_lp, c_pert, c_count, c_tmp;
  // gradient: chunk buffers, block sums, coefficients
  DBuf g_h1, g_h2, g_g, g_gz2, g_gz1, g_x, g_ones, g_bsum, g_w1, g_w2, g_w3, g_b, g_coef, g_mean, g_part, g_flag, g_out,
      g_keys, g_w, g_loc;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  // SR: selection, Jacobian rows, stacked matrix, Gram eigensystem
  DBuf s_lpk, s_lpk2, s_idx, s_idx2, s_keys, s_sw, s_R, s_mean, s_S, s_gram, s_w, s_t, s_u, s_dir, s_boff, s_info,
      s_work, s_grad, s_coef1, s_tmp;
  // device-resident flat parameters (AnqsModel::params) and Adam state (optimizer.cpp:17-31)
  DBuf theta, adam_m, adam_v, adam_d, adam_bad, p_boff;
  long adam_t = 0;
  // fill_amplitudes of the sampler's own batch (qvmc_cuda_fill_amplitudes): parameter version,
  // the last sampled batch's size / version and device fingerprints [sample, fill]
  uint64_t params_version = 0, samp_version = ~uint64_t{0};
  int64_t samp_n = -1;
  bool fast_fill = true;   // QVMC_FAST_FILL=0: always evaluate both heads
  int last_fill_sampled = 0;
  DBuf fpb;
  // the phase heads' activations of the last sampled-batch fill, for the gradient of that batch
  // (QVMC_GRAD_CACHE=0 disables): rows, parameter version, keys fingerprint
  DBuf hcache;
  bool grad_cache = true;
  int64_t hc_n = -1;
  uint64_t hc_version = ~uint64_t{0};
  unsigned long long hc_fp = 0;
  int last_grad_cached = 0;
  ~qvmc_model_s() {
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
  }
};

namespace {
void check_model(qvmc_model_s* m) {
  if (!m) fail(QVMC_ERR_INVALID_ARGUMENT, "null model handle");
}

int64_t model_param_count(int n, int bits, int hidden) {
  int64_t c = 0;
  for (int o = 0; o < n; o += bits) {
    const int out = 1 << std::min(bits, n - o);
    c += 2 * (static_cast<int64_t>(hidden) * n + hidden + static_cast<int64_t>(hidden) * hidden + hidden +
              static_cast<int64_t>(out) * hidden + out);
  }
  return c;
}

// half_lp != null: the batch is the sampler's own (log|psi| = 0.5 log p), only the phase heads run
void launch_log_psi(qvmc_model_s* m, const uint64_t* keys, int64_t n, double* la, double* ph,
                    const double* half_lp = nullptr, double* hcache = nullptr) {
  if (n == 0) return;
  using namespace qvmc_model;
  ModelView V{m->P.as<double>(), m->n, m->n_qudits, m->bits, m->n_e, m->spin, m->n_up};
  if (!m->tiled && !half_lp) {  // CTA-per-sample-tile kernel (all qudits in one CTA)
    const int grid = static_cast<int>((n + kTile - 1) / kTile);
    const size_t dyn = static_cast<size_t>((1 + kWBufs) * kHid * kTile) * sizeof(double);
    DISPATCH_W(m->W, {
      ck(cudaFuncSetAttribute(k_log_psi<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)),
         "smem attribute");
      k_log_psi<WW><<<grid, kMThreads, dyn, m->stream>>>(V, keys, n, la, ph);
    });
    ck_launch("log_psi");
    return;
  }
  // warp-tiled: CTAs = (qudit, head) blocks x sample chunks, sized to whole waves of 148 SMs
  const int n_jh = half_lp ? m->n_qudits : 2 * m->n_qudits;
  const int64_t max_chunks = std::max<int64_t>(1, (n + kWT * kPWarps - 1) / (kWT * kPWarps));
  int64_t best_s = 1;
  double best_eff = -1.0;
  for (int w = 4; w <= 16; ++w) {
    const int64_t S = std::min<int64_t>(max_chunks, std::max<int64_t>(1, (int64_t{m->sms} * w) / n_jh));
    const int64_t blocks = S * n_jh;
    const int64_t waves = (blocks + m->sms - 1) / m->sms;
    const double eff = static_cast<double>(blocks) / static_cast<double>(waves * m->sms) + 1e-3 * w;
    if (eff > best_eff) {
      best_eff = eff;
      best_s = S;
    }
  }
  int64_t chunk = (n + best_s - 1) / best_s;
  chunk = (chunk + kWT - 1) / kWT * kWT;
  const int64_t S = (n + chunk - 1) / chunk;
  m->part.ensure(static_cast<size_t>(2 * m->n_qudits) * n * sizeof(double));
  DISPATCH_W(m->W, {
    const size_t dyn = (8448 + kPWarps * 64 * kWT) * sizeof(double) + kPWarps * kWT * WW * sizeof(uint64_t);
    ck(cudaFuncSetAttribute(k_log_psi_part<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)),
       "smem attribute");
    k_log_psi_part<WW><<<static_cast<unsigned>(S * n_jh), kPThreads, dyn, m->stream>>>(
        V, keys, n, chunk, m->part.as<double>(), -1, nullptr, half_lp ? 1 : 0, half_lp ? hcache : nullptr);
    ck_launch("log_psi part");
    if (half_lp)
      k_sum_phases<WW><<<static_cast<unsigned>((n + 255) / 256), 256, 0, m->stream>>>(V, keys, n, m->part.as<double>(),
                                                                                     half_lp, la, ph);
    else
      k_sum_qudits<WW><<<static_cast<unsigned>((n + 255) / 256), 256, 0, m->stream>>>(V, keys, n,
                                                                                    m->part.as<double>(), la, ph);
    ck_launch("log_psi sum");
  });
}
}  // namespace

extern "C" {

int qvmc_cuda_model_create(int n_qubits, int bits_per_qudit, int n_electrons, int spin_constraint, int hidden,
                           int device, qvmc_model_t* out) {
  return guarded([&] {
    if (!out) fail(QVMC_ERR_INVALID_ARGUMENT, "null output handle");
    // QuditLayout::make (model.cpp:33-37), AnqsModel::AnqsModel (model.cpp:49-58)
    if (n_qubits < 1 || n_qubits > 256) fail(QVMC_ERR_INVALID_ARGUMENT, "QuditLayout: qubit count out of range");
    if (bits_per_qudit < 1 || bits_per_qudit > 8)
      fail(QVMC_ERR_INVALID_ARGUMENT, "QuditLayout: bits_per_qudit must be in [1, 8]");
    if (n_electrons < 0 || n_electrons > n_qubits) fail(QVMC_ERR_INVALID_ARGUMENT, "AnqsModel: electron count out of range");
    if (spin_constraint && n_electrons % 2 != 0)
      fail(QVMC_ERR_INVALID_ARGUMENT, "AnqsModel: spin constraint requires even n_electrons");
    if (hidden < 1) fail(QVMC_ERR_INVALID_ARGUMENT, "AnqsModel: hidden width must be positive");
    if (hidden != qvmc_model::kHid || bits_per_qudit > qvmc_model::kMaxK)
      fail(QVMC_ERR_INVALID_ARGUMENT, "device amplitude path supports hidden = 64 and bits_per_qudit <= 6");
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) fail(QVMC_ERR_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= n_dev) fail(QVMC_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    DeviceGuard dg(device);
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) fail(QVMC_ERR_NO_DEVICE, "libqvmc_cuda is built for sm_100a (B200) only");
    auto m = std::make_unique<qvmc_model_s>();
    m->device = device;
    m->n = n_qubits;
    m->W = (n_qubits + 63) / 64;
    m->bits = bits_per_qudit;
    m->n_e = n_electrons;
    m->spin = spin_constraint ? 1 : 0;
    m->n_up = spin_constraint ? n_electrons / 2 : 0;
    m->hidden = hidden;
    m->n_qudits = (n_qubits + bits_per_qudit - 1) / bits_per_qudit;
    m->n_params = model_param_count(n_qubits, bits_per_qudit, hidden);
    m->sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("QVMC_MODEL_TILED")) m->tiled = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_FAST_FILL")) m->fast_fill = std::atoi(e) != 0;
    if (const char* e = std::getenv("QVMC_GRAD_CACHE")) m->grad_cache = std::atoi(e) != 0;
    ck(cudaStreamCreateWithFlags(&m->own, cudaStreamNonBlocking), "stream create");
    m->stream = m->own;
    *out = m.release();
  });
}

int qvmc_cuda_model_destroy(qvmc_model_t m) {
  return guarded([&] {
    if (!m) return;
    DeviceGuard dg(m->device);
    if (m->own) {
      cudaStreamSynchronize(m->own);
      cudaStreamDestroy(m->own);
    }
    delete m;
  });
}

int qvmc_cuda_model_n_params(qvmc_model_t m, int64_t* out) {
  return guarded([&] {
    check_model(m);
    if (!out) fail(QVMC_ERR_INVALID_ARGUMENT, "null output");
    *out = m->n_params;
  });
}

int qvmc_cuda_model_set_stream(qvmc_model_t m, void* stream) {
  return guarded([&] {
    check_model(m);
    m->stream = stream ? static_cast<cudaStream_t>(stream) : m->own;
  });
}

// AnqsModel::set_params (model.cpp:99-103): host vector in the reference's flat
// layout (model.cpp:65-80); re-laid out for the kernel and uploaded.
int qvmc_cuda_model_set_params(qvmc_model_t m, int64_t n_params, const double* params) {
  return guarded([&] {
    check_model(m);
    if (n_params != m->n_params) fail(QVMC_ERR_INVALID_ARGUMENT, "AnqsModel::set_params: size mismatch");
    if (!params) fail(QVMC_ERR_INVALID_ARGUMENT, "null params");
    using namespace qvmc_model;
    const int n = m->n, H = kHid;
    const BlockLayout L{n};
    std::vector<double> dev(static_cast<size_t>(m->n_qudits) * 2 * L.size(), 0.0);
    int64_t cur = 0;
    for (int j = 0; j < m->n_qudits; ++j) {
      const int off = j * m->bits, k = std::min(m->bits, n - off), out = 1 << k;
      for (int hd = 0; hd < 2; ++hd) {
        const double* w1 = params + cur;
        const double* b1 = w1 + static_cast<int64_t>(H) * n;
        const double* w2 = b1 + H;
        const double* b2 = w2 + H * H;
        const double* w3 = b2 + H;
        const double* b3 = w3 + out * H;
        cur += static_cast<int64_t>(H) * n + H + H * H + H + out * H + out;
        double* B = dev.data() + static_cast<size_t>(2 * j + hd) * L.size();
        for (int h = 0; h < H; ++h) {
          double c = 0.0;
          for (int i = 0; i < n; ++i) {
            B[L.w1t() + i * H + h] = w1[static_cast<int64_t>(h) * n + i];
            if (i < off) c += w1[static_cast<int64_t>(h) * n + i];
          }
          B[L.csum() + h] = c;
          B[L.b1() + h] = b1[h];
          B[L.b2() + h] = b2[h];
          for (int kk = 0; kk < H; ++kk) B[L.w2t() + kk * H + h] = w2[h * H + kk];
        }
        for (int v = 0; v < out; ++v) {
          B[L.b3() + v] = b3[v];
          for (int kk = 0; kk < H; ++kk) B[L.w3t() + kk * H + v] = w3[v * H + kk];
        }
      }
    }
    if (cur != m->n_params) fail(QVMC_ERR_RUNTIME, "parameter layout mismatch");
    DeviceGuard dg(m->device);
    m->P.ensure(dev.size() * sizeof(double));
    ck(cudaMemcpyAsync(m->P.p, dev.data(), dev.size() * sizeof(double), cudaMemcpyHostToDevice, m->stream), "H2D params");
    m->theta.ensure(m->n_params * 8);  // the flat vector stays on the device too (Adam, get_params)
    ck(cudaMemcpyAsync(m->theta.p, params, m->n_params * 8, cudaMemcpyHostToDevice, m->stream), "H2D theta");
    ck(cudaStreamSynchronize(m->stream), "sync");  // the host staging vector goes out of scope
    m->has_params = true;
    ++m->params_version;
  });
}

// sample_without_replacement (sampler.cpp:37-102) on the device; see
// qvmc_sampler.cuh. Returns the batch size; the keys and log-probabilities are
// in the reference's ChildLess order.
int qvmc_cuda_sample(qvmc_model_t m, int k_samples, uint64_t seed, uint32_t stream, uint32_t iteration, int mem,
                     uint64_t* out_keys, double* out_log_probs, int64_t* out_n) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (k_samples < 1) fail(QVMC_ERR_INVALID_ARGUMENT, "sample_without_replacement: K must be >= 1");
    if (k_samples > (1 << 25)) fail(QVMC_ERR_INVALID_ARGUMENT, "sample_without_replacement: K above 2^25");
    if (!out_keys || !out_log_probs || !out_n) fail(QVMC_ERR_INVALID_ARGUMENT, "null output");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    using namespace qvmc_model;
    using namespace qvmc_sampler;
    DeviceGuard dg(m->device);
    const int W = m->W;
    const int64_t K = k_samples;
    const size_t maxc = static_cast<size_t>(K) * 64;
    for (int i = 0; i < 2; ++i) {
      m->bk[i].ensure(K * W * 8 + 16);
      m->blp[i].ensure(K * 8 + 16);
      m->bpert[i].ensure(K * 8 + 16);
    }
    m->cond.ensure(K * 64 * 8 + 16);
    m->c_key.ensure(maxc * 8 + 16);
    m->c_key2.ensure(maxc * 8 + 16);
    m->c_slot.ensure(maxc * 4 + 16);
    m->c_slot2.ensure(maxc * 4 + 16);
    m->c_bv.ensure(maxc * 4 + 16);
    m->c_lp.ensure(maxc * 8 + 16);
    m->c_pert.ensure(maxc * 8 + 16);
    m->c_count.ensure(16);
    {  // CUB temporary storage for the largest possible candidate count, once (no growth mid-call)
      size_t tb_max = 0;
      ck(cub::DeviceRadixSort::SortPairs(nullptr, tb_max, m->c_key.as<uint64_t>(), m->c_key2.as<uint64_t>(),
                                         m->c_slot.as<uint32_t>(), m->c_slot2.as<uint32_t>(),
                                         static_cast<int>(std::min<size_t>(maxc, 0x7FFFFFFF)), 0, 64, m->stream),
         "sort size");
      m->c_tmp.ensure(tb_max + 16);
    }
    // root: the empty prefix, log p = 0, perturbed = 0 (sampler.cpp:45-46)
    ck(cudaMemsetAsync(m->bk[0].p, 0, W * 8, m->stream), "memset");
    ck(cudaMemsetAsync(m->blp[0].p, 0, 8, m->stream), "memset");
    ck(cudaMemsetAsync(m->bpert[0].p, 0, 8, m->stream), "memset");
    int cur = 0;
    int64_t B = 1;
    ModelView V{m->P.as<double>(), m->n, m->n_qudits, m->bits, m->n_e, m->spin, m->n_up};
    Candidates Cd{m->c_key.as<uint64_t>(), m->c_slot.as<uint32_t>(), m->c_bv.as<uint32_t>(), m->c_lp.as<double>(),
                  m->c_pert.as<double>(), m->c_count.as<unsigned long long>()};
    const bool trace = std::getenv("QVMC_SAMPLER_TRACE") != nullptr;
    cudaEvent_t tev[6];
    if (trace)
      for (auto& e : tev) ck(cudaEventCreate(&e), "event");
    for (int level = 0; level < m->n_qudits; ++level) {
      const int off = level * m->bits, k = std::min(m->bits, m->n - off);
      if (trace) ck(cudaEventRecord(tev[0], m->stream), "event");
      // 1. conditional log-probabilities of every beam prefix (amplitude head of this qudit)
      const int64_t per = static_cast<int64_t>(kWT) * kPWarps;
      const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>((B + per - 1) / per, 4 * m->sms));
      int64_t chunk = (B + chunks - 1) / chunks;
      chunk = (chunk + kWT - 1) / kWT * kWT;
      const int64_t S = (B + chunk - 1) / chunk;
      DISPATCH_W(W, {
        const size_t dyn = (8448 + kPWarps * 64 * kWT) * sizeof(double) + kPWarps * kWT * WW * sizeof(uint64_t);
        ck(cudaFuncSetAttribute(k_log_psi_part<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(dyn)), "smem attribute");
        k_log_psi_part<WW><<<static_cast<unsigned>(S), kPThreads, dyn, m->stream>>>(
            V, m->bk[cur].as<uint64_t>(), B, chunk, nullptr, level, m->cond.as<double>());
        ck_launch("sampler conditional");
      });
      // 2. children + Gumbel + condition_max
      if (trace) ck(cudaEventRecord(tev[1], m->stream), "event");
      ck(cudaMemsetAsync(m->c_count.p, 0, 8, m->stream), "memset");
      const int eg = static_cast<int>(std::min<int64_t>((B * 32 + 255) / 256, 8LL * m->sms));
      k_expand<<<std::max(eg, 1), 256, 0, m->stream>>>(m->cond.as<double>(), m->blp[cur].as<double>(),
                                                        m->bpert[cur].as<double>(), B, 1 << k, seed, stream,
                                                        iteration, static_cast<uint32_t>(level), Cd);
      ck_launch("sampler expand");
      unsigned long long nc = 0;
      ck(cudaMemcpyAsync(&nc, m->c_count.p, 8, cudaMemcpyDeviceToHost, m->stream), "D2H count");
      ck(cudaStreamSynchronize(m->stream), "sync");
      if (nc == 0) fail(QVMC_ERR_RUNTIME, "sample_without_replacement: empty sector");
      // 3. ChildLess order: conditioned value descending, ties by child prefix
      if (trace) ck(cudaEventRecord(tev[2], m->stream), "event");
      const int n = static_cast<int>(nc);
      size_t tb = 0;
      ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, m->c_key.as<uint64_t>(), m->c_key2.as<uint64_t>(),
                                         m->c_slot.as<uint32_t>(), m->c_slot2.as<uint32_t>(), n, 0, 64, m->stream),
         "sort size");
      m->c_tmp.ensure(tb + 16);
      ck(cub::DeviceRadixSort::SortPairs(m->c_tmp.p, tb, m->c_key.as<uint64_t>(), m->c_key2.as<uint64_t>(),
                                         m->c_slot.as<uint32_t>(), m->c_slot2.as<uint32_t>(), n, 0, 64, m->stream),
         "sort");
      ++g_launches;
      const int64_t keep = std::min<int64_t>(K, n);
      const int tg = static_cast<int>(std::min<int64_t>((keep + 255) / 256, 8LL * m->sms));
      if (trace) ck(cudaEventRecord(tev[3], m->stream), "event");
      DISPATCH_W(W, {
        k_ties<WW><<<std::max(tg, 1), 256, 0, m->stream>>>(m->c_key2.as<uint64_t>(), m->c_slot2.as<uint32_t>(), n,
                                                          keep, m->c_bv.as<uint32_t>(), m->bk[cur].as<uint64_t>(),
                                                          off, k);
        ck_launch("sampler ties");
        // 4. the next beam
        k_gather_beam<WW><<<std::max(tg, 1), 256, 0, m->stream>>>(
            m->c_slot2.as<uint32_t>(), keep, Cd, m->bk[cur].as<uint64_t>(), off, k, m->bk[1 - cur].as<uint64_t>(),
            m->blp[1 - cur].as<double>(), m->bpert[1 - cur].as<double>());
        ck_launch("sampler gather");
      });
      if (trace) {
        ck(cudaEventRecord(tev[4], m->stream), "event");
        ck(cudaEventSynchronize(tev[4]), "sync");
        float t[4];
        for (int q = 0; q < 4; ++q) ck(cudaEventElapsedTime(&t[q], tev[q], tev[q + 1]), "elapsed");
        std::fprintf(stderr, "sampler level %d: beam %lld candidates %llu | cond %.3f expand+count %.3f sort %.3f "
                     "ties+gather %.3f ms\n", level, static_cast<long long>(B), nc, t[0], t[1], t[2], t[3]);
      }
      cur = 1 - cur;
      B = keep;
    }
    if (trace)
      for (auto& e : tev) cudaEventDestroy(e);
    const cudaMemcpyKind kind = mem == QVMC_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    ck(cudaMemcpyAsync(out_keys, m->bk[cur].p, B * W * 8, kind, m->stream), "copy keys");
    ck(cudaMemcpyAsync(out_log_probs, m->blp[cur].p, B * 8, kind, m->stream), "copy log_probs");
    // fingerprint of this batch: fill_amplitudes recognises it and halves its log p (k_sum_phases)
    m->fpb.ensure(4 * sizeof(unsigned long long));
    ck(cudaMemsetAsync(m->fpb.p, 0, sizeof(unsigned long long), m->stream), "memset fingerprint");
    if (B > 0)
      DISPATCH_W(W, (qvmc_model::k_fingerprint<WW><<<static_cast<unsigned>(std::min<int64_t>((B + 255) / 256,
                                                                                             4 * m->sms)),
                                                     256, 0, m->stream>>>(m->bk[cur].as<uint64_t>(),
                                                                          m->blp[cur].as<double>(), B,
                                                                          m->fpb.as<unsigned long long>())));
    ck(cudaStreamSynchronize(m->stream), "sync");
    *out_n = B;
    m->samp_n = B;
    m->samp_version = m->params_version;
  });
}

}  // extern "C"

namespace {

void blas_ck(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS) fail(QVMC_ERR_CUDA, std::string(what) + ": cuBLAS status " + std::to_string(st));
}

template <int W>
__global__ void k_sector_flags(const uint64_t* __restrict__ keys, int64_t n, int n_e, int spin, int n_up,
                               int* __restrict__ bad) {
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int pc = 0, pe = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint64_t x = keys[s * W + w];
      pc += __popcll(x);
      pe += __popcll(x & 0x5555555555555555ull);
    }
    if (pc != n_e || (spin && pe != n_up)) atomicOr(bad, 1);
  }
}

// forward (h1, h2, coefficient-scaled g) then backward (gz2, gz1) kernels of the gradient
// into the chunk buffers (block stride n_blk rows)
template <int W>
void launch_grad_parts(qvmc_model_s* m, const qvmc_model::ModelView& V, const uint64_t* keys, int64_t n, int64_t per,
                       int64_t S, int nb, const double2* coef, int64_t n_blk, const double* hc = nullptr,
                       int64_t hc_rows = 0) {
  using namespace qvmc_model;
  const size_t dyn_f = (8448 + kG2Warps * 64 * kWT + kG2Warps * 64) * sizeof(double) +
                       kG2Warps * kWT * W * sizeof(uint64_t);
  const size_t dyn_b = (8192 + kG2Warps * 64 * kWT + kG2Warps * 64) * sizeof(double);
  m->g_bsum.ensure(static_cast<size_t>(2 * S * nb) * 64 * sizeof(double));  // Σ g, Σ gz2 per (block, CTA)
  ck(cudaFuncSetAttribute(k_grad_fwd<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn_f)),
     "smem attribute");
  ck(cudaFuncSetAttribute(k_grad_bwd<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn_b)),
     "smem attribute");
  k_grad_fwd<W><<<static_cast<unsigned>(S * nb), kG2Threads, dyn_f, m->stream>>>(
      V, keys, n, per, coef, m->g_h1.as<double>(), m->g_h2.as<double>(), m->g_g.as<double>(), n_blk,
      m->g_bsum.as<double>(), hc, hc_rows);
  ck_launch("grad forward");
  k_grad_bwd<W><<<static_cast<unsigned>(S * nb), kG2Threads, dyn_b, m->stream>>>(
      V, keys, n, per, m->g_h1.as<double>(), m->g_h2.as<double>(), m->g_g.as<double>(), m->g_gz2.as<double>(),
      m->g_gz1.as<double>(), n_blk, m->g_bsum.as<double>() + static_cast<size_t>(S * nb) * 64);
  ck_launch("grad backward");
}

// Σ over samples of coefficient-scaled gradient blocks (k_grad_fwd / k_grad_bwd + strided-batched DGEMMs)
// into m->g_w1/g_w2/g_w3/g_b; coef [n] device (2 Re c, 2 Im c); keys device
void grad_accumulate(qvmc_model_s* m, const uint64_t* keys, int64_t n, const double2* coef) {
  using namespace qvmc_model;
  const int nb = 2 * m->n_qudits, nq = m->n, W = m->W, nx = nq + 2;
  ModelView V{m->P.as<double>(), m->n, m->n_qudits, m->bits, m->n_e, m->spin, m->n_up};
  if (!m->blas) blas_ck(cublasCreate(&m->blas), "cublasCreate");
  blas_ck(cublasSetStream(m->blas, m->stream), "cublasSetStream");
  // the batch of the last sampled-batch fill under the current parameters (same size, version and keys
  // fingerprint): its phase blocks copy the cached activations instead of recomputing them
  bool cached = false;
  if (m->hc_n == n && n > 0 && m->hc_version == m->params_version) {
    m->fpb.ensure(4 * sizeof(unsigned long long));
    ck(cudaMemsetAsync(m->fpb.as<unsigned long long>() + 3, 0, sizeof(unsigned long long), m->stream), "memset");
    DISPATCH_W(W, (k_fingerprint<WW><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4 * m->sms)), 256, 0,
                                       m->stream>>>(keys, nullptr, n, m->fpb.as<unsigned long long>() + 3)));
    ck_launch("keys fingerprint");
    unsigned long long fp = 0;
    ck(cudaMemcpyAsync(&fp, m->fpb.as<unsigned long long>() + 3, 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
    cached = fp == m->hc_fp;
  }
  m->last_grad_cached = cached ? 1 : 0;
  // split-K: every chunk's sample range is cut into `parts` slices so the
  // batched GEMMs (64 x 64 outputs, one per block) fill the SMs; partial sums
  // are added in part order by k_sum_parts (deterministic)
  const int parts = nb <= 24 ? 16 : 8;
  const int64_t Nc = std::min<int64_t>(std::max<int64_t>(n, 1), 32768);
  const int64_t Kp_max = ((Nc + parts - 1) / parts + 7) / 8 * 8;
  const int64_t Ncp = Kp_max * parts;  // padded chunk rows
  m->g_h1.ensure(static_cast<size_t>(nb) * Ncp * 64 * 8);
  m->g_h2.ensure(static_cast<size_t>(nb) * Ncp * 64 * 8);
  m->g_g.ensure(static_cast<size_t>(nb) * Ncp * 64 * 8);
  m->g_gz2.ensure(static_cast<size_t>(nb) * Ncp * 64 * 8);
  m->g_gz1.ensure(static_cast<size_t>(nb) * Ncp * 64 * 8);
  m->g_x.ensure(static_cast<size_t>(Ncp) * nx * 8);
  const size_t l1 = static_cast<size_t>(64) * nx, l2 = static_cast<size_t>(64) * kHS;
  m->g_ones.ensure(static_cast<size_t>(nb) * parts * std::max(l1, l2) * 8);  // split-K partials (reused)
  m->g_w1.ensure(static_cast<size_t>(nb) * l1 * 8);
  m->g_w2.ensure(static_cast<size_t>(nb) * l2 * 8);
  m->g_w3.ensure(static_cast<size_t>(nb) * l2 * 8);
  const double one = 1.0, zero = 0.0;
  // pointer arrays of the W1 GEMMs (X is shared by the blocks, so its slice depends on the part only);
  // they depend on the chunk geometry alone: one set for full chunks, one for the last, uploaded once
  // (no host round trip between chunks)
  const size_t np = static_cast<size_t>(nb) * parts;
  m->s_tmp.ensure(np * 6 * sizeof(void*) + 16);
  {
    std::vector<void*> ptrs(np * 6);
    const int64_t last = n - (n > 0 ? (n - 1) / Nc * Nc : 0);
    for (int set = 0; set < 2; ++set) {
      const int64_t nc = set == 0 ? Nc : last;
      const int64_t Kp = ((nc + parts - 1) / parts + 7) / 8 * 8;
      const int64_t Ncur = Kp * parts;
      void** pp = ptrs.data() + set * np * 3;
      for (int jh = 0; jh < nb; ++jh)
        for (int q = 0; q < parts; ++q) {
          const size_t b2 = static_cast<size_t>(jh) * parts + q;
          pp[b2] = m->g_x.as<double>() + q * Kp * nx;
          pp[np + b2] = m->g_gz1.as<double>() + (static_cast<int64_t>(jh) * Ncur + q * Kp) * 64;
          pp[2 * np + b2] = m->g_ones.as<double>() + b2 * l1;
        }
    }
    ck(cudaMemcpyAsync(m->s_tmp.p, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice, m->stream),
       "H2D ptrs");
    ck(cudaStreamSynchronize(m->stream), "sync");  // the host vector goes out of scope
  }
  for (int64_t c0 = 0; c0 < n; c0 += Nc) {
    const int64_t nc = std::min<int64_t>(Nc, n - c0);
    const int64_t Kp = ((nc + parts - 1) / parts + 7) / 8 * 8;
    const int64_t Ncur = Kp * parts;  // this chunk's padded rows: rows >= nc must be zero
    if (Ncur > nc) {
      ck(cudaMemsetAsync(m->g_h1.p, 0, static_cast<size_t>(nb) * Ncur * 64 * 8, m->stream), "memset");
      ck(cudaMemsetAsync(m->g_h2.p, 0, static_cast<size_t>(nb) * Ncur * 64 * 8, m->stream), "memset");
      ck(cudaMemsetAsync(m->g_g.p, 0, static_cast<size_t>(nb) * Ncur * 64 * 8, m->stream), "memset");
      ck(cudaMemsetAsync(m->g_gz2.p, 0, static_cast<size_t>(nb) * Ncur * 64 * 8, m->stream), "memset");
      ck(cudaMemsetAsync(m->g_gz1.p, 0, static_cast<size_t>(nb) * Ncur * 64 * 8, m->stream), "memset");
      ck(cudaMemsetAsync(m->g_x.p, 0, static_cast<size_t>(Ncur) * nx * 8, m->stream), "memset");
    }
    const int64_t per = 1024;  // samples per CTA
    const int64_t S = (nc + per - 1) / per;
    DISPATCH_W(W, {
      launch_grad_parts<WW>(m, V, keys + c0 * WW, nc, per, S, nb, coef + c0, Ncur,
                            cached ? m->hcache.as<double>() + c0 * 128 : nullptr, n);
      const int xg = static_cast<int>(std::min<int64_t>((nc * nx + 255) / 256, 8LL * m->sms));
      k_pm_bits<WW><<<xg, 256, 0, m->stream>>>(keys + c0 * WW, nc, nq, m->g_x.as<double>());
      ck_launch("pm bits");
    });
    const int first = c0 == 0 ? 1 : 0;
    double* part = m->g_ones.as<double>();
    // gW2 / gW3 (+ gb2 / gb3 in row 64): batch b = jh * parts + p, A = H[b * Kp rows], B = vectors[b * Kp rows]
    // W2 / W3: M = 64 (the h rows carry no bias column); the bias rows (64) come from the kernels' sums
    const int n_cta = static_cast<int>((nc + 1023) / 1024);
    const int bgrid = static_cast<int>(std::min<int64_t>((nb * parts * 64 + 255) / 256, 1024));
    blas_ck(cublasDgemmStridedBatched(m->blas, CUBLAS_OP_N, CUBLAS_OP_T, 64, 64, static_cast<int>(Kp), &one,
                                      m->g_h1.as<double>(), 64, Kp * 64, m->g_gz2.as<double>(), 64, Kp * 64,
                                      &zero, part, kHS, static_cast<long long>(l2), nb * parts), "dgemm w2");
    k_bias_rows<<<bgrid, 256, 0, m->stream>>>(m->g_bsum.as<double>() + static_cast<size_t>(n_cta) * nb * 64, nb,
                                              n_cta, parts, static_cast<int64_t>(l2), part);
    k_sum_parts<<<static_cast<int>(std::min<size_t>((nb * l2 + 255) / 256, 4096)), 256, 0, m->stream>>>(
        part, nb, parts, static_cast<int64_t>(l2), first, m->g_w2.as<double>());
    blas_ck(cublasDgemmStridedBatched(m->blas, CUBLAS_OP_N, CUBLAS_OP_T, 64, 64, static_cast<int>(Kp), &one,
                                      m->g_h2.as<double>(), 64, Kp * 64, m->g_g.as<double>(), 64, Kp * 64,
                                      &zero, part, kHS, static_cast<long long>(l2), nb * parts), "dgemm w3");
    k_bias_rows<<<bgrid, 256, 0, m->stream>>>(m->g_bsum.as<double>(), nb, n_cta, parts, static_cast<int64_t>(l2),
                                              part);
    k_sum_parts<<<static_cast<int>(std::min<size_t>((nb * l2 + 255) / 256, 4096)), 256, 0, m->stream>>>(
        part, nb, parts, static_cast<int64_t>(l2), first, m->g_w3.as<double>());
    // gW1 (+ gb1 in row n): pointer-array batch, X slice by part
    void** dp = static_cast<void**>(m->s_tmp.p) + (nc == Nc ? 0 : np * 3);
    blas_ck(cublasDgemmBatched(m->blas, CUBLAS_OP_N, CUBLAS_OP_T, nx, 64, static_cast<int>(Kp), &one,
                               reinterpret_cast<const double* const*>(dp), nx,
                               reinterpret_cast<const double* const*>(dp + np), 64, &zero,
                               reinterpret_cast<double* const*>(dp + 2 * np), nx, nb * parts), "dgemm w1");
    k_sum_parts<<<static_cast<int>(std::min<size_t>((nb * l1 + 255) / 256, 4096)), 256, 0, m->stream>>>(
        part, nb, parts, static_cast<int64_t>(l1), first, m->g_w1.as<double>());
    ck_launch("split-K sums");
    g_launches += 7;
  }
}

// flat offsets of the (qudit, head) parameter blocks (model.cpp:65-80), nb + 1 entries
std::vector<int64_t> block_offsets(const qvmc_model_s* m) {
  std::vector<int64_t> b(1, 0);
  for (int jh = 0; jh < 2 * m->n_qudits; ++jh) {
    const int k = std::min(m->bits, m->n - (jh >> 1) * m->bits);
    b.push_back(b.back() + 64LL * m->n + 64 + 4096 + 64 + (64LL << k) + (1 << k));
  }
  return b;
}

void solver_ck(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS) fail(QVMC_ERR_CUDA, std::string(what) + ": cuSOLVER status " + std::to_string(st));
}

__global__ void k_iota_u32(uint32_t* p, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<uint32_t>(i);
}

__global__ void k_gather_rows_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx, int64_t n, int W,
                                  uint64_t* __restrict__ dst) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * W;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[e] = src[static_cast<int64_t>(idx[e / W]) * W + e % W];
}

// sr_direction (sr.cpp:74-95) on device buffers: S row-major [rows][cols] (= col-major cols x rows),
// grad [cols] -> out [cols]; lambda > 0. The Gram eigensystem is cuSOLVER syevd.
void sr_solve_device(qvmc_model_s* m, int64_t rows, int64_t cols, const double* S, double lambda, const double* grad,
                     double* out) {
  if (!m->blas) blas_ck(cublasCreate(&m->blas), "cublasCreate");
  if (!m->solver) solver_ck(cusolverDnCreate(&m->solver), "cusolverDnCreate");
  blas_ck(cublasSetStream(m->blas, m->stream), "cublasSetStream");
  solver_ck(cusolverDnSetStream(m->solver, m->stream), "cusolverDnSetStream");
  const int r = static_cast<int>(rows), c = static_cast<int>(cols);
  const double one = 1.0, zero = 0.0, mone = -1.0;
  m->s_gram.ensure(static_cast<size_t>(r) * r * 8 + 16);
  m->s_w.ensure(static_cast<size_t>(r) * 8 + 16);
  m->s_t.ensure(static_cast<size_t>(r) * 8 + 16);
  m->s_u.ensure(static_cast<size_t>(r) * 8 + 16);
  m->s_info.ensure(16);
  double* gram = m->s_gram.as<double>();
  // gram = S S^T + lambda I   (S^T S in col-major terms of the c x r matrix)
  blas_ck(cublasDgemm(m->blas, CUBLAS_OP_T, CUBLAS_OP_N, r, r, c, &one, S, c, S, c, &zero, gram, r), "dgemm gram");
  {
    std::vector<double> eye(static_cast<size_t>(r), lambda);
    m->s_tmp.ensure(static_cast<size_t>(r) * 8 + 16);
    ck(cudaMemcpyAsync(m->s_tmp.p, eye.data(), r * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
    blas_ck(cublasDaxpy(m->blas, r, &one, m->s_tmp.as<double>(), 1, gram, r + 1), "daxpy diag");
    ck(cudaStreamSynchronize(m->stream), "sync");
  }
  int lwork = 0;
  solver_ck(cusolverDnDsyevd_bufferSize(m->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r, gram, r,
                                        m->s_w.as<double>(), &lwork), "syevd size");
  m->s_work.ensure(static_cast<size_t>(lwork) * 8 + 16);
  solver_ck(cusolverDnDsyevd(m->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r, gram, r,
                             m->s_w.as<double>(), m->s_work.as<double>(), lwork, m->s_info.as<int>()), "syevd");
  int info = 0;
  std::vector<double> ev(static_cast<size_t>(r));
  ck(cudaMemcpyAsync(&info, m->s_info.p, 4, cudaMemcpyDeviceToHost, m->stream), "D2H");
  ck(cudaMemcpyAsync(ev.data(), m->s_w.p, r * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
  ck(cudaStreamSynchronize(m->stream), "sync");
  if (info != 0) fail(QVMC_ERR_RUNTIME, "sr_direction: eigendecomposition failed");
  const double lo = *std::min_element(ev.begin(), ev.end()), hi = *std::max_element(ev.begin(), ev.end());
  if (!(lo > 0.0) || hi / lo > 1e14) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", hi / std::max(lo, 1e-300));
    fail(QVMC_ERR_RUNTIME, std::string("sr_direction: ill-conditioned system, cond ~ ") + buf);
  }
  // t = S grad; u = (V^T t) ./ evals; s = V u; out = (grad - S^T s) / lambda
  blas_ck(cublasDgemv(m->blas, CUBLAS_OP_T, c, r, &one, S, c, grad, 1, &zero, m->s_t.as<double>(), 1), "gemv t");
  blas_ck(cublasDgemv(m->blas, CUBLAS_OP_T, r, r, &one, gram, r, m->s_t.as<double>(), 1, &zero,
                      m->s_u.as<double>(), 1), "gemv u");
  {
    std::vector<double> inv(static_cast<size_t>(r));
    for (int i = 0; i < r; ++i) inv[i] = 1.0 / ev[i];
    ck(cudaMemcpyAsync(m->s_tmp.p, inv.data(), r * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
    blas_ck(cublasDdgmm(m->blas, CUBLAS_SIDE_LEFT, r, 1, m->s_u.as<double>(), r, m->s_tmp.as<double>(), 1,
                        m->s_u.as<double>(), r), "ddgmm");
    ck(cudaStreamSynchronize(m->stream), "sync");
  }
  blas_ck(cublasDgemv(m->blas, CUBLAS_OP_N, r, r, &one, gram, r, m->s_u.as<double>(), 1, &zero,
                      m->s_t.as<double>(), 1), "gemv s");
  ck(cudaMemcpyAsync(out, grad, static_cast<size_t>(c) * 8, cudaMemcpyDeviceToDevice, m->stream), "copy grad");
  blas_ck(cublasDgemv(m->blas, CUBLAS_OP_N, c, r, &mone, S, c, m->s_t.as<double>(), 1, &one, out, 1), "gemv out");
  const double il = 1.0 / lambda;
  blas_ck(cublasDscal(m->blas, c, &il, out, 1), "dscal");
  g_launches += 8;
}

void check_in_sector(qvmc_model_s* m, const uint64_t* keys, int64_t n) {
  m->g_flag.ensure(16);
  ck(cudaMemsetAsync(m->g_flag.p, 0, 4, m->stream), "memset");
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 8LL * m->sms));
  DISPATCH_W(m->W, (k_sector_flags<WW><<<std::max(grid, 1), 256, 0, m->stream>>>(keys, n, m->n_e, m->spin, m->n_up,
                                                                                   m->g_flag.as<int>())));
  ck_launch("sector flags");
  int bad = 0;
  ck(cudaMemcpyAsync(&bad, m->g_flag.p, 4, cudaMemcpyDeviceToHost, m->stream), "D2H");
  ck(cudaStreamSynchronize(m->stream), "sync");
  if (bad) fail(QVMC_ERR_INVALID_ARGUMENT, "grad_log_psi: state is masked (zero amplitude)");
}

}  // namespace

extern "C" {

// energy_gradient (energy.cpp:93-107) with batched_grad_log_psi rows (model.cpp:273-336)
// contracted on the device, never materialised.
int qvmc_cuda_energy_gradient(qvmc_model_t m, int64_t n, const uint64_t* keys, const double* weights,
                              const double* locals, int mem, double* out_grad) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (n < 1) fail(QVMC_ERR_INVALID_ARGUMENT, "energy_gradient: misaligned inputs");
    if (!keys || !weights || !locals || !out_grad) fail(QVMC_ERR_INVALID_ARGUMENT, "null array");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    using namespace qvmc_model;
    DeviceGuard dg(m->device);
    const uint64_t* dk = keys;
    const double* dw = weights;
    const double2* dl = reinterpret_cast<const double2*>(locals);
    if (mem == QVMC_MEM_HOST) {
      m->g_keys.ensure(n * m->W * 8);
      m->g_w.ensure(n * 8);
      m->g_loc.ensure(n * 16);
      ck(cudaMemcpyAsync(m->g_keys.p, keys, n * m->W * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      ck(cudaMemcpyAsync(m->g_w.p, weights, n * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      ck(cudaMemcpyAsync(m->g_loc.p, locals, n * 16, cudaMemcpyHostToDevice, m->stream), "H2D");
      dk = m->g_keys.as<uint64_t>();
      dw = m->g_w.as<double>();
      dl = m->g_loc.as<double2>();
    }
    check_in_sector(m, dk, n);
    m->g_part.ensure(kLseBlocks * 16);
    m->g_mean.ensure(16);
    m->g_coef.ensure(n * 16);
    k_wmean_partial<<<kLseBlocks, 256, 0, m->stream>>>(dw, dl, n, m->g_part.as<double2>());
    k_wmean_final<<<1, 32, 0, m->stream>>>(m->g_part.as<double2>(), kLseBlocks, m->g_mean.as<double2>());
    const int cg = static_cast<int>(std::min<int64_t>((n + 255) / 256, 8LL * m->sms));
    k_grad_coef<<<cg, 256, 0, m->stream>>>(dw, dl, n, m->g_mean.as<double2>(), m->g_coef.as<double2>());
    ck_launch("gradient coefficients");
    g_launches += 2;
    grad_accumulate(m, dk, n, m->g_coef.as<double2>());
    ModelView V{m->P.as<double>(), m->n, m->n_qudits, m->bits, m->n_e, m->spin, m->n_up};
    double* dout = out_grad;
    if (mem == QVMC_MEM_HOST) {
      m->g_out.ensure(m->n_params * 8);
      dout = m->g_out.as<double>();
    }
    k_grad_scatter<<<2 * m->n_qudits, 256, 0, m->stream>>>(V, m->g_w1.as<double>(), m->g_w2.as<double>(),
                                                            m->g_w3.as<double>(), dout);
    ck_launch("gradient scatter");
    if (mem == QVMC_MEM_HOST)
      ck(cudaMemcpyAsync(out_grad, dout, m->n_params * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
  });
}

// sr_direction (sr.cpp:74-95) for a given stacked matrix (SrContext::stacked,
// row-major [rows][cols] here) and lambda > 0.
int qvmc_cuda_sr_solve(qvmc_model_t m, int64_t rows, int64_t cols, const double* stacked, double lambda,
                       const double* grad, int mem, double* out_direction) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (rows < 1 || cols < 1 || rows > 65536 || cols > (1LL << 31) / std::max<int64_t>(rows, 1))
      fail(QVMC_ERR_INVALID_ARGUMENT, "sr_direction: bad system size");
    if (!stacked || !grad || !out_direction) fail(QVMC_ERR_INVALID_ARGUMENT, "null array");
    if (!(lambda > 0.0)) fail(QVMC_ERR_INVALID_ARGUMENT, "sr_direction: lambda must be positive");
    DeviceGuard dg(m->device);
    const double* dS = stacked;
    const double* dg2 = grad;
    double* dout = out_direction;
    if (mem == QVMC_MEM_HOST) {
      m->s_S.ensure(static_cast<size_t>(rows) * cols * 8);
      m->s_grad.ensure(static_cast<size_t>(cols) * 8);
      m->s_dir.ensure(static_cast<size_t>(cols) * 8);
      ck(cudaMemcpyAsync(m->s_S.p, stacked, rows * cols * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      ck(cudaMemcpyAsync(m->s_grad.p, grad, cols * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      dS = m->s_S.as<double>();
      dg2 = m->s_grad.as<double>();
      dout = m->s_dir.as<double>();
    }
    sr_solve_device(m, rows, cols, dS, lambda, dg2, dout);
    if (mem == QVMC_MEM_HOST)
      ck(cudaMemcpyAsync(out_direction, dout, cols * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
  });
}

// The SR step of run_optimisation (optimizer.cpp:105-143) on the device:
// top_probability_indices (sr.cpp:15-23) -> grad_log_psi rows of the selected
// samples -> build_sr_context (sr.cpp:25-72) -> sr_direction (sr.cpp:74-95).
int qvmc_cuda_sr_direction(qvmc_model_t m, int64_t n, const uint64_t* keys, const double* log_probs,
                           const double* locals, int n_sr, double lambda, const double* grad, int mem,
                           double* out_direction, double* out_lambda) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (n < 1 || n_sr < 1) fail(QVMC_ERR_INVALID_ARGUMENT, "build_sr_context: empty selection");
    if (!keys || !log_probs || !locals || !grad || !out_direction) fail(QVMC_ERR_INVALID_ARGUMENT, "null array");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    using namespace qvmc_model;
    DeviceGuard dg(m->device);
    const int W = m->W;
    const int64_t P = m->n_params, ns = std::min<int64_t>(n_sr, n);
    const uint64_t* dk = keys;
    const double *dlp = log_probs, *dgr = grad;
    (void)locals;  // sr_direction's context needs the samples and weights only (sr.cpp:25-72)
    if (mem == QVMC_MEM_HOST) {
      m->g_keys.ensure(n * W * 8);
      m->g_w.ensure(n * 8);
      m->s_grad.ensure(P * 8);
      ck(cudaMemcpyAsync(m->g_keys.p, keys, n * W * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      ck(cudaMemcpyAsync(m->g_w.p, log_probs, n * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      ck(cudaMemcpyAsync(m->s_grad.p, grad, P * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      dk = m->g_keys.as<uint64_t>();
      dlp = m->g_w.as<double>();
      dgr = m->s_grad.as<double>();
    }
    // 1. top_probability_indices: stable sort by log p descending (ties keep sample order)
    m->s_lpk.ensure(n * 8 + 16);
    m->s_lpk2.ensure(n * 8 + 16);
    m->s_idx.ensure(n * 4 + 16);
    m->s_idx2.ensure(n * 4 + 16);
    k_iota_u32<<<std::max(1, static_cast<int>(std::min<int64_t>((n + 255) / 256, 4096))), 256, 0, m->stream>>>(
        m->s_idx.as<uint32_t>(), n);
    ck_launch("iota");
    ck(cudaMemcpyAsync(m->s_lpk.p, dlp, n * 8, cudaMemcpyDeviceToDevice, m->stream), "copy lp");
    size_t tb = 0;
    ck(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, m->s_lpk.as<double>(), m->s_lpk2.as<double>(),
                                                 m->s_idx.as<uint32_t>(), m->s_idx2.as<uint32_t>(),
                                                 static_cast<int>(n), 0, 64, m->stream), "sort size");
    m->s_work.ensure(tb + 16);
    ck(cub::DeviceRadixSort::SortPairsDescending(m->s_work.p, tb, m->s_lpk.as<double>(), m->s_lpk2.as<double>(),
                                                 m->s_idx.as<uint32_t>(), m->s_idx2.as<uint32_t>(),
                                                 static_cast<int>(n), 0, 64, m->stream), "sort");
    ++g_launches;
    std::vector<uint32_t> sel(static_cast<size_t>(ns));
    std::vector<double> slp(static_cast<size_t>(ns));
    ck(cudaMemcpyAsync(sel.data(), m->s_idx2.p, ns * 4, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaMemcpyAsync(slp.data(), m->s_lpk2.p, ns * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
    // 2. weights re-renormalised over the subset, Ē (sr.cpp:36-53), gathered keys
    double mx = slp[0];
    for (double v : slp) mx = std::max(mx, v);
    std::vector<double> w(static_cast<size_t>(ns)), sw(static_cast<size_t>(ns));
    double sum = 0.0;
    for (int64_t i = 0; i < ns; ++i) sum += (w[i] = std::exp(slp[i] - mx));
    for (int64_t i = 0; i < ns; ++i) {
      w[i] /= sum;
      sw[i] = std::sqrt(w[i]);
    }
    m->s_keys.ensure(ns * W * 8 + 16);
    k_gather_rows_u64<<<std::max(1, static_cast<int>(std::min<int64_t>((ns * W + 255) / 256, 4096))), 256, 0,
                        m->stream>>>(dk, m->s_idx2.as<uint32_t>(), ns, W, m->s_keys.as<uint64_t>());
    ck_launch("gather keys");
    check_in_sector(m, m->s_keys.as<uint64_t>(), ns);
    // 3. Jacobian rows R [ns][P] (k_grad_fwd / k_grad_bwd with coefficients (1, 1), then the outer products)
    m->s_coef1.ensure(ns * 16 + 16);
    {
      std::vector<double> ones(static_cast<size_t>(2 * ns), 1.0);
      ck(cudaMemcpyAsync(m->s_coef1.p, ones.data(), ns * 16, cudaMemcpyHostToDevice, m->stream), "H2D");
    }
    const int nb = 2 * m->n_qudits, nq = m->n;
    const size_t vb = static_cast<size_t>(nb) * ns * 64 * 8;
    m->g_h1.ensure(static_cast<size_t>(nb) * ns * 64 * 8);
    m->g_h2.ensure(static_cast<size_t>(nb) * ns * 64 * 8);
    m->g_g.ensure(vb);
    m->g_gz2.ensure(vb);
    m->g_gz1.ensure(vb);
    m->g_x.ensure(static_cast<size_t>(ns) * (nq + 2) * 8);
    ModelView V{m->P.as<double>(), m->n, m->n_qudits, m->bits, m->n_e, m->spin, m->n_up};
    const auto boff = block_offsets(m);
    m->s_boff.ensure(boff.size() * 8);
    ck(cudaMemcpyAsync(m->s_boff.p, boff.data(), boff.size() * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
    DISPATCH_W(W, {
      const int64_t per = 1024, S = (ns + per - 1) / per;
      launch_grad_parts<WW>(m, V, m->s_keys.as<uint64_t>(), ns, per, S, nb, m->s_coef1.as<double2>(), ns);
      k_pm_bits<WW><<<std::max(1, static_cast<int>(std::min<int64_t>((ns * (nq + 2) + 255) / 256, 4096))), 256, 0,
                      m->stream>>>(m->s_keys.as<uint64_t>(), ns, nq, m->g_x.as<double>());
      ck_launch("sr pm bits");
    });
    m->s_R.ensure(static_cast<size_t>(ns) * P * 8);
    k_jac_real<<<dim3(static_cast<unsigned>(ns), nb), 256, 0, m->stream>>>(
        V, m->s_boff.as<int64_t>(), ns, m->g_h1.as<double>(), m->g_h2.as<double>(), m->g_g.as<double>(),
        m->g_gz2.as<double>(), m->g_gz1.as<double>(), m->g_x.as<double>(), P, m->s_R.as<double>());
    ck_launch("jacobian rows");
    // 4. mean row, stacked [2 ns][P]
    if (!m->blas) blas_ck(cublasCreate(&m->blas), "cublasCreate");
    blas_ck(cublasSetStream(m->blas, m->stream), "cublasSetStream");
    m->s_sw.ensure(ns * 16 + 16);
    ck(cudaMemcpyAsync(m->s_sw.p, w.data(), ns * 8, cudaMemcpyHostToDevice, m->stream), "H2D w");
    ck(cudaMemcpyAsync(m->s_sw.as<double>() + ns, sw.data(), ns * 8, cudaMemcpyHostToDevice, m->stream), "H2D sw");
    m->s_mean.ensure(P * 8);
    const double one = 1.0, zero = 0.0;
    blas_ck(cublasDgemv(m->blas, CUBLAS_OP_N, static_cast<int>(P), static_cast<int>(ns), &one, m->s_R.as<double>(),
                        static_cast<int>(P), m->s_sw.as<double>(), 1, &zero, m->s_mean.as<double>(), 1), "gemv mean");
    m->s_S.ensure(static_cast<size_t>(2 * ns) * P * 8);
    k_sr_stack<<<dim3(static_cast<unsigned>(ns), nb), 256, 0, m->stream>>>(
        V, m->s_boff.as<int64_t>(), ns, m->s_R.as<double>(), m->s_mean.as<double>(), m->s_sw.as<double>() + ns, P,
        m->s_S.as<double>());
    ck_launch("sr stack");
    // 5. lambda: given, or 1e-4 (1 + ||stacked||_F^2 / n_sr) (sr.cpp:68-71)
    double lam = lambda;
    if (!(lam > 0.0)) {
      double nrm = 0.0;
      blas_ck(cublasSetPointerMode(m->blas, CUBLAS_POINTER_MODE_HOST), "pointer mode");
      blas_ck(cublasDnrm2(m->blas, static_cast<int>(2 * ns * P), m->s_S.as<double>(), 1, &nrm), "dnrm2");
      lam = 1e-4 * (1.0 + nrm * nrm / static_cast<double>(ns));
    }
    double* dout = out_direction;
    if (mem == QVMC_MEM_HOST) {
      m->s_dir.ensure(P * 8);
      dout = m->s_dir.as<double>();
    }
    sr_solve_device(m, 2 * ns, P, m->s_S.as<double>(), lam, dgr, dout);
    if (mem == QVMC_MEM_HOST) ck(cudaMemcpyAsync(out_direction, dout, P * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
    if (out_lambda) *out_lambda = lam;
  });
}

// AnqsModel::params() (model.hpp:66): the flat vector, host or device copy.
int qvmc_cuda_model_get_params(qvmc_model_t m, int mem, double* out) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (!out) fail(QVMC_ERR_INVALID_ARGUMENT, "null output");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    DeviceGuard dg(m->device);
    ck(cudaMemcpyAsync(out, m->theta.p, m->n_params * 8,
                       mem == QVMC_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, m->stream), "copy");
    ck(cudaStreamSynchronize(m->stream), "sync");
  });
}

// adam_step (optimizer.cpp:17-31) + model.set_params(theta) (optimizer.cpp:157) with
// the parameters, the Adam state (created zero on first use) and the kernels' layout
// all on the device.
int qvmc_cuda_model_adam_step(qvmc_model_t m, const double* direction, double learning_rate, double beta1,
                              double beta2, double epsilon, int mem) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (!direction) fail(QVMC_ERR_INVALID_ARGUMENT, "null direction");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    using namespace qvmc_model;
    DeviceGuard dg(m->device);
    const int64_t P = m->n_params;
    if (m->adam_m.bytes < static_cast<size_t>(P) * 8) {
      m->adam_m.ensure(P * 8);
      m->adam_v.ensure(P * 8);
      ck(cudaMemsetAsync(m->adam_m.p, 0, P * 8, m->stream), "memset");
      ck(cudaMemsetAsync(m->adam_v.p, 0, P * 8, m->stream), "memset");
      m->adam_t = 0;
    }
    const double* dd = direction;
    if (mem == QVMC_MEM_HOST) {
      m->adam_d.ensure(P * 8);
      ck(cudaMemcpyAsync(m->adam_d.p, direction, P * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
      dd = m->adam_d.as<double>();
    }
    m->adam_bad.ensure(16);
    ck(cudaMemsetAsync(m->adam_bad.p, 0, 4, m->stream), "memset");
    const int grid = static_cast<int>(std::min<int64_t>((P + 255) / 256, 8LL * m->sms));
    k_adam_check<<<grid, 256, 0, m->stream>>>(dd, P, m->adam_bad.as<int>());
    ck_launch("adam check");
    const long t = m->adam_t + 1;
    const double c1 = 1.0 - std::pow(beta1, static_cast<double>(t)), c2 = 1.0 - std::pow(beta2, static_cast<double>(t));
    k_adam<<<grid, 256, 0, m->stream>>>(dd, P, learning_rate, beta1, beta2, epsilon, c1, c2, m->adam_bad.as<int>(),
                                        m->adam_m.as<double>(), m->adam_v.as<double>(), m->theta.as<double>());
    ck_launch("adam");
    int bad = 0;
    ck(cudaMemcpyAsync(&bad, m->adam_bad.p, 4, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
    if (bad) fail(QVMC_ERR_RUNTIME, "adam_step: non-finite direction entry");
    m->adam_t = t;
    const auto boff = block_offsets(m);
    m->p_boff.ensure(boff.size() * 8);
    ck(cudaMemcpyAsync(m->p_boff.p, boff.data(), boff.size() * 8, cudaMemcpyHostToDevice, m->stream), "H2D");
    ModelView V{m->P.as<double>(), m->n, m->n_qudits, m->bits, m->n_e, m->spin, m->n_up};
    k_params_relayout<<<2 * m->n_qudits, 256, 0, m->stream>>>(V, m->p_boff.as<int64_t>(), m->theta.as<double>(),
                                                              m->P.as<double>());
    ck_launch("params relayout");
    ++m->params_version;
    ck(cudaStreamSynchronize(m->stream), "sync");
  });
}

// AnqsModel::log_psi (model.cpp:262-271) for every key: the loop of
// fill_amplitudes (sampler.cpp:104-112).
int qvmc_cuda_log_psi(qvmc_model_t m, int64_t n, const uint64_t* keys, int mem, double* out_log_amp,
                      double* out_phase) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (n < 0) fail(QVMC_ERR_INVALID_ARGUMENT, "negative batch size");
    if (n > 0 && (!keys || !out_log_amp || !out_phase)) fail(QVMC_ERR_INVALID_ARGUMENT, "null array");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    DeviceGuard dg(m->device);
    const uint64_t* dk = keys;
    double *dla = out_log_amp, *dph = out_phase;
    if (mem == QVMC_MEM_HOST) {
      m->keys.ensure(std::max<size_t>(n * m->W * 8, 16));
      m->la.ensure(std::max<size_t>(n * 8, 16));
      m->ph.ensure(std::max<size_t>(n * 8, 16));
      if (n) ck(cudaMemcpyAsync(m->keys.p, keys, n * m->W * 8, cudaMemcpyHostToDevice, m->stream), "H2D keys");
      dk = m->keys.as<uint64_t>();
      dla = m->la.as<double>();
      dph = m->ph.as<double>();
    }
    launch_log_psi(m, dk, n, dla, dph);
    if (mem == QVMC_MEM_HOST) {
      if (n) {
        ck(cudaMemcpyAsync(out_log_amp, dla, n * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
        ck(cudaMemcpyAsync(out_phase, dph, n * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
      }
      ck(cudaStreamSynchronize(m->stream), "sync");
    }
  });
}

// fill_amplitudes (sampler.cpp:104-120): log_psi of every key plus
// (norm, log_norm) = logsumexp of the sampler's log_probs. out_norm2 is a host
// pointer in either memory kind (the call synchronises).
int qvmc_cuda_fill_amplitudes(qvmc_model_t m, int64_t n, const uint64_t* keys, const double* log_probs, int mem,
                              double* out_log_amp, double* out_phase, double* out_norm2) {
  return guarded([&] {
    check_model(m);
    check_mem(mem);
    if (n < 0) fail(QVMC_ERR_INVALID_ARGUMENT, "negative batch size");
    if ((n > 0 && !log_probs) || !out_norm2) fail(QVMC_ERR_INVALID_ARGUMENT, "null array");
    if (n == 0) {  // sampler.cpp:114-119 over no samples: log_norm = -inf + log(0), norm = 0
      out_norm2[0] = 0.0;
      out_norm2[1] = -std::numeric_limits<double>::infinity();
      return;
    }
    if (!keys || !out_log_amp || !out_phase) fail(QVMC_ERR_INVALID_ARGUMENT, "null array");
    if (!m->has_params) fail(QVMC_ERR_INVALID_ARGUMENT, "model parameters not set");
    DeviceGuard dg(m->device);
    const uint64_t* dk = keys;
    const double* dlp = log_probs;
    double *dla = out_log_amp, *dph = out_phase;
    if (mem == QVMC_MEM_HOST) {
      m->keys.ensure(std::max<size_t>(n * m->W * 8, 16));
      m->la.ensure(std::max<size_t>(n * 8, 16));
      m->ph.ensure(std::max<size_t>(n * 8, 16));
      m->lp.ensure(n * 8);
      ck(cudaMemcpyAsync(m->keys.p, keys, n * m->W * 8, cudaMemcpyHostToDevice, m->stream), "H2D keys");
      ck(cudaMemcpyAsync(m->lp.p, log_probs, n * 8, cudaMemcpyHostToDevice, m->stream), "H2D log_probs");
      dk = m->keys.as<uint64_t>();
      dlp = m->lp.as<double>();
      dla = m->la.as<double>();
      dph = m->ph.as<double>();
    }
    // the batch qvmc_cuda_sample produced under the current parameters (same size and version,
    // same fingerprint of keys and log p): log|psi| = 0.5 log p exactly, phase heads only
    bool sampled = false;
    if (m->fast_fill && m->tiled && n == m->samp_n && m->params_version == m->samp_version) {
      ck(cudaMemsetAsync(m->fpb.as<unsigned long long>() + 1, 0, sizeof(unsigned long long), m->stream), "memset");
      DISPATCH_W(m->W, (qvmc_model::k_fingerprint<WW><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256,
                                                                                                4 * m->sms)),
                                                        256, 0, m->stream>>>(dk, dlp, n,
                                                                             m->fpb.as<unsigned long long>() + 1)));
      ck_launch("fingerprint");
      unsigned long long fp[2] = {0, 0};
      ck(cudaMemcpyAsync(fp, m->fpb.p, sizeof(fp), cudaMemcpyDeviceToHost, m->stream), "D2H fingerprints");
      ck(cudaStreamSynchronize(m->stream), "sync");
      sampled = fp[0] == fp[1];
    }
    m->last_fill_sampled = sampled ? 1 : 0;
    // keep the phase heads' activations for the gradient of this batch (at most 48 GB)
    const size_t hc_bytes = static_cast<size_t>(m->n_qudits) * static_cast<size_t>(n) * 128 * sizeof(double);
    const bool keep = sampled && m->grad_cache && hc_bytes <= (size_t{48} << 30);
    m->hc_n = -1;
    if (keep) {
      m->hcache.ensure(hc_bytes);
      ck(cudaMemsetAsync(m->fpb.as<unsigned long long>() + 2, 0, sizeof(unsigned long long), m->stream), "memset");
      DISPATCH_W(m->W, (qvmc_model::k_fingerprint<WW><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256,
                                                                                                4 * m->sms)),
                                                        256, 0, m->stream>>>(dk, nullptr, n,
                                                                             m->fpb.as<unsigned long long>() + 2)));
      ck_launch("keys fingerprint");
    }
    launch_log_psi(m, dk, n, dla, dph, sampled ? dlp : nullptr, keep ? m->hcache.as<double>() : nullptr);
    using namespace qvmc_model;
    m->lse.ensure(kLseBlocks * sizeof(double2));
    m->out2.ensure(2 * sizeof(double));
    k_lse_partial<<<kLseBlocks, 256, 0, m->stream>>>(dlp, n, m->lse.as<double2>());
    ck_launch("lse partial");
    k_lse_final<<<1, 32, 0, m->stream>>>(m->lse.as<double2>(), kLseBlocks, m->out2.as<double>());
    ck_launch("lse final");
    if (mem == QVMC_MEM_HOST) {
      ck(cudaMemcpyAsync(out_log_amp, dla, n * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
      ck(cudaMemcpyAsync(out_phase, dph, n * 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    }
    ck(cudaMemcpyAsync(out_norm2, m->out2.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->stream), "D2H norm");
    unsigned long long kfp = 0;
    if (keep) ck(cudaMemcpyAsync(&kfp, m->fpb.as<unsigned long long>() + 2, 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
    ck(cudaStreamSynchronize(m->stream), "sync");
    if (keep) {
      m->hc_n = n;
      m->hc_version = m->params_version;
      m->hc_fp = kfp;
    }
  });
}

// 1 when the last qvmc_cuda_fill_amplitudes recognised the sampler's own batch (phase heads only)
int qvmc_cuda_model_last_fill_sampled(qvmc_model_t m) { return m ? m->last_fill_sampled : 0; }

// 1 when the last qvmc_cuda_energy_gradient reused the sampled-batch fill's phase-head activations
int qvmc_cuda_model_last_gradient_cached(qvmc_model_t m) { return m ? m->last_grad_cached : 0; }

int qvmc_cuda_model_synchronize(qvmc_model_t m) {
  return guarded([&] {
    check_model(m);
    DeviceGuard dg(m->device);
    ck(cudaStreamSynchronize(m->stream), "sync");
  });
}

}  // extern "C"
