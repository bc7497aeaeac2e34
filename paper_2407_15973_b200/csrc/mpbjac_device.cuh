// mpbjac_device.cuh — device helpers shared by the libmpbjac kernels.
//
// Built with --fmad=false (see Makefile): every a*b+c below is two IEEE
// roundings, exactly like the reference's numba/numpy arithmetic
// (pkg/src/mpcg/kernels_numba.py:1-13: fastmath off).  Division and sqrt are
// the IEEE-rounded defaults (no -use_fast_math).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mpbjac_order.h"

namespace mpb {

constexpr int kTileThreads = MPB_TILE_THREADS;  // lanes of the tile sum order
constexpr int kTileRows = MPB_TILE_MAX_ROWS;
constexpr int kCtaThreads = kTileRows;           // tile kernels: one thread per row
constexpr int kFinThreads = MPB_FIN_THREADS;
static_assert(kTileRows == kTileThreads, "one lane of the tile sum per row");

// ---------------------------------------------------------------------------
// solver state (device resident; one per solve)
// ---------------------------------------------------------------------------
enum SolveError {
  kOk = 0,
  kBreakdown = 1,
  kIndefPrecond = 2,
  kIndefMatrix = 3,
  kNonFinite = 4,
  kNarrowOverflow = 5
};

struct SolverState {
  // scalars of the recurrence (solver.py:133-169)
  double rho, rho_prev, pq, alpha, beta, rnorm, relres, r0;
  double res_tol, adp_tol;
  double final_true;
  double err_val;
  long long it;       // iteration in progress (1-based)
  long long last_it;  // iteration whose trace entry was written last
  long long cap;
  long long stride;
  long long err_it;
  unsigned long long t0_ns;
  unsigned long long ovf_count;
  long long ovf_first;
  // trace arrays (device, cap entries each)
  double *tr_relres;
  double *tr_true;
  int *tr_branch;
  double *tr_time;
  unsigned int ticket[4];  // last-CTA counters of the fused scalar steps
  double red_local[2];     // multi-GPU: this rank's sum (and overflow count)
  double red_global[2];    //            after the all-reduce
  int dist;                // multi-GPU: scalar steps wait for the all-reduce
  int kind;
  int branch;  // 0 high (fp64 instance), 1 low (fp32 instance)
  int first;   // p is None (solver.py:150-151)
  int done;
  int converged;
  int error;
  int true_pending;
  int z1_ok;       // the fused update already ran the next first pass for `branch`
  int upd_branch;  // branch of the iteration whose x/r update is pending (set at kStepPq)
  int wave_epoch;  // wave kernels completed in this solve (their group counters' target)
  unsigned long long cond;  // while-node handle of the solve graph (0: host-polled loop)
  unsigned long long *tl;   // diagnostics (MPB_TIMELINE): per-iteration kernel timestamps, or null
};

// MPB_TIMELINE: tl[(it % kTlIters) * kTlStride + kind * 4 + f], kind 0 last pass,
// 1 SpMV, 2 fused update; f 0 first consumer start, 1 last consumer end,
// 2 scalar step (globaltimer ns)
constexpr int kTlIters = 1024;
constexpr int kTlStride = 16;  // kinds 0-2 as above; kind 3: last-pass CTA entry min / max, post-wait max
__device__ __forceinline__ unsigned long long globaltimer_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// compiled in only with -DMPB_TIMELINE (make EXTRA=-DMPB_TIMELINE): the
// extra state load sits on the critical path of warp 0
__device__ __forceinline__ void tl_mark(const SolverState *st, int kind, int f, bool is_max) {
#ifndef MPB_TIMELINE
  return;
#endif
  if (st == nullptr || st->tl == nullptr) return;
  unsigned long long *p = st->tl + (st->it % kTlIters) * kTlStride + kind * 4 + f;
  const unsigned long long t = globaltimer_now();
  if (is_max) atomicMax(p, t); else atomicMin(p, t);
}
// the same with a time taken earlier (e.g. at CTA entry, before st->it is final)
__device__ __forceinline__ void tl_mark_at(const SolverState *st, int kind, int f, bool is_max, unsigned long long t) {
#ifndef MPB_TIMELINE
  return;
#endif
  if (st == nullptr || st->tl == nullptr) return;
  unsigned long long *p = st->tl + (st->it % kTlIters) * kTlStride + kind * 4 + f;
  if (is_max) atomicMax(p, t); else atomicMin(p, t);
}

// ---------------------------------------------------------------------------
// reductions in the order fixed by include/mpbjac_order.h
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_bfly(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_bfly(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Two butterflies at once (a lane's values of two 32-row groups): after the
// xor-16 level lanes 0-15 carry the first value's partial sums and lanes
// 16-31 the second's (a + b computed by one of the two lanes that would both
// compute it -- IEEE addition commutes), and the remaining levels stay inside
// the 16-lane halves.  Every sum is formed from the same operands as in
// warp_bfly, so the totals are bit-identical: lanes 0-15 return v0's, lanes
// 16-31 v1's.  One shuffle per level instead of two.
__device__ __forceinline__ double warp_bfly2(double v0, double v1) {
  const bool hi = (threadIdx.x & 16) != 0;
  const double send = hi ? v0 : v1, keep = hi ? v1 : v0;
  double v = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16));
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Steps 2-3: per-warp butterfly then warp 0 butterflies the warp sums padded
// with +0 to 32 lanes.  Result valid in thread 0.  ws: 32 entries of smem.
template <int NT, typename R>
__device__ __forceinline__ R block_tree(R v, R *ws) {
  static_assert(NT % 32 == 0 && NT <= 1024, "block size");
  v = warp_bfly(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  R r = R(0);
  if (warp == 0) {
    r = lane < NT / 32 ? ws[lane] : R(0);
    r = warp_bfly(r);
  }
  return r;
}

// Named barrier among the first `n` threads (consumer warps of a
// warp-specialised CTA; the producer warp does not take part).
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// block_tree over the first NT threads using named barrier `bar`.
template <int NT, typename R>
__device__ __forceinline__ R block_tree_nb(R v, R *ws, int bar) {
  static_assert(NT % 32 == 0 && NT <= 1024, "block size");
  v = warp_bfly(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  named_sync(bar, NT);
  if (lane == 0) ws[warp] = v;
  named_sync(bar, NT);
  R r = R(0);
  if (warp == 0) {
    r = lane < NT / 32 ? ws[lane] : R(0);
    r = warp_bfly(r);
  }
  return r;
}

// Global sum of tile partials, steps 1-3 with kFinThreads lanes.  Called by
// all threads of a CTA; RPT lanes per thread (lanes t + k * kFinThreads/RPT,
// for CTAs with fewer than kFinThreads compute threads), threads beyond
// contribute nothing; result valid in thread 0.  Partials are read through
// L2 (__ldcg): other SMs wrote them in the same kernel.
// B: loads in flight per lane (16 halves the L2 round trips of 8; kernels
// whose register budget it would raise keep 8)
template <int B = 16, int RPT = 1>
__device__ __forceinline__ double fin_sum(const double *part, long long count, double *ws) {
  constexpr int NT = kFinThreads / RPT;
  double acc[RPT];
#pragma unroll
  for (int k = 0; k < RPT; k++) acc[k] = 0.0;
  if (threadIdx.x < NT) {
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      for (long long i0 = threadIdx.x + k * NT; i0 < count; i0 += (long long)B * kFinThreads) {
        double v[B];
#pragma unroll
        for (int u = 0; u < B; u++) {
          const long long i = i0 + (long long)u * kFinThreads;
          v[u] = i < count ? __ldcg(part + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; u++)
          if (i0 + (long long)u * kFinThreads < count) acc[k] = __dadd_rn(acc[k], v[u]);
      }
    }
  }
  if (RPT == 1) return block_tree<kFinThreads>(acc[0], ws);
  // virtual warps (lane t + k NT), then warp 0 over the kFinThreads/32 warp sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < RPT; k++) acc[k] = warp_bfly(acc[k]);
  __syncthreads();
  if (lane == 0 && threadIdx.x < NT) {
#pragma unroll
    for (int k = 0; k < RPT; k++) ws[warp + k * (NT / 32)] = acc[k];
  }
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < kFinThreads / 32 ? ws[lane] : 0.0;
    r = warp_bfly(r);
  }
  return r;
}

// ---- two-level global sums (include/mpbjac_order.h) -------------------------
constexpr int kChunkTiles = MPB_CHUNK_TILES;
static_assert(kChunkTiles == 8 * 32, "a chunk sum is one warp emulating 8 warps of 32 lanes");

// C_c = the tile-sum order over chunk c's partials (lane j of 256 holds
// P[c*256 + j] or +0), computed by one warp: the 8 virtual warps'
// butterflies, then the butterfly of their sums padded with +0.  All lanes
// return C_c.  Partials written by other CTAs in this kernel: read via L2.
template <typename R>
__device__ __forceinline__ R chunk_sum_warp(const R *part, long long c, long long ntiles) {
  const int lane = threadIdx.x & 31;
  const long long base = c * kChunkTiles;
  R v[kChunkTiles / 32];
#pragma unroll
  for (int w = 0; w < kChunkTiles / 32; w++) {
    const long long i = base + 32 * w + lane;
    v[w] = i < ntiles ? __ldcg(part + i) : R(0);
  }
#pragma unroll
  for (int w = 0; w < kChunkTiles / 32; w++) v[w] = warp_bfly(v[w]);
  R r = R(0);
#pragma unroll
  for (int w = 0; w < kChunkTiles / 32; w++)
    if (lane == w) r = v[w];
  return warp_bfly(r);
}

// Chunk sums while the kernel runs, without per-tile fences: a tile partial
// is its own completion flag.  The partials array holds kPartEmpty (all
// bits set, a NaN no tile sum is stored as) in every slot between kernels;
// a tile's partial is one 8-byte relaxed store; the warp that owns chunk c
// (the CTA that claimed the chunk's last tile) polls the chunk's slots with
// relaxed loads until none is empty, sums them (chunk_sum order), stores
// csum[c] and empties the slots for the next launch.  The kernel's final
// CTA reads csum after the grid ticket (acq_rel).
constexpr unsigned long long kPartEmpty = ~0ull;
__device__ __forceinline__ void put_part(double *p, double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  if (b == kPartEmpty) b = 0x7ff8000000000000ull;  // (still a NaN; the empty pattern stays unique)
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}
__device__ __forceinline__ unsigned long long get_part_bits(const double *p) {
  unsigned long long b;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  return b;
}

// Two-level sums only above MPB_ONE_LEVEL_TILES tiles (include/mpbjac_order.h).
__host__ __device__ inline bool two_level(long long ntiles) { return ntiles > MPB_ONE_LEVEL_TILES; }

struct ChunkCtx {
  double *csum;  // null: no chunk bookkeeping (plugin-level launch)
  double *part;
  int ntiles;
  int poll;      // two-level order: chunk owners poll (two_level(ntiles))
};
__device__ __forceinline__ bool chunk_final(int tile, int ntiles) {
  return tile % kChunkTiles == kChunkTiles - 1 || tile == ntiles - 1;
}
// One warp; chunk c's slots polled once (block: until complete).  On
// completion the chunk sum is stored and the slots emptied; returns whether
// it completed.
__device__ __forceinline__ bool chunk_poll(const ChunkCtx &ck, int c, bool block) {
  const int lane = threadIdx.x & 31;
  const int base = c * kChunkTiles + lane;  // (tile indices are int32)
  const double *pb = ck.part + base;
  const int lim = ck.ntiles - base;         // slot w is a tile iff 32 w < lim
  for (;;) {
    unsigned long long b[kChunkTiles / 32];
    bool full = true;
#pragma unroll
    for (int w = 0; w < kChunkTiles / 32; w++) {
      b[w] = 32 * w < lim ? get_part_bits(pb + 32 * w) : 0ull;  // (+0.0 beyond the last tile)
      full = full && b[w] != kPartEmpty;
    }
    if (__all_sync(0xffffffffu, full)) {
      double v[kChunkTiles / 32];
#pragma unroll
      for (int w = 0; w < kChunkTiles / 32; w++) v[w] = warp_bfly(__longlong_as_double(static_cast<long long>(b[w])));
      double r = 0.0;
#pragma unroll
      for (int w = 0; w < kChunkTiles / 32; w++)
        if (lane == w) r = v[w];
      r = warp_bfly(r);
      if (lane == 0) ck.csum[c] = r;
#pragma unroll
      for (int w = 0; w < kChunkTiles / 32; w++)
        if (32 * w < lim) reinterpret_cast<unsigned long long *>(const_cast<double *>(pb))[32 * w] = kPartEmpty;
      return true;
    }
    if (!block) return false;
    __nanosleep(200);
  }
}

// All chunks by the CTA that took the grid's last ticket, warps taking
// chunks round-robin (two-level kernels whose grid may exceed residency, so
// that no CTA may wait for another); the slots are emptied.  Called by all
// threads.
__device__ __forceinline__ void chunk_all_in_cta(const ChunkCtx &ck) {
  if (ck.csum == nullptr) return;
  const int nch = (ck.ntiles + kChunkTiles - 1) / kChunkTiles;
  for (int c = threadIdx.x >> 5; c < nch; c += blockDim.x >> 5) {
    const double v = chunk_sum_warp(static_cast<const double *>(ck.part), c, ck.ntiles);
    if ((threadIdx.x & 31) == 0) ck.csum[c] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ck.ntiles; i += blockDim.x) reinterpret_cast<unsigned long long *>(ck.part)[i] = kPartEmpty;
  __syncthreads();
}

// Non-warp-specialised persistent kernels (static walk tile0, tile0 +
// stride, ...): after its tiles, warp 0 owns the chunks whose last tile it
// processed.  Called by all threads.
__device__ __forceinline__ void chunk_duties_strided(const ChunkCtx &ck, int tile0, int stride) {
  if (ck.csum == nullptr || !ck.poll) return;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  for (int t = tile0; t < ck.ntiles; t += stride)
    if (chunk_final(t, ck.ntiles)) chunk_poll(ck, t / kChunkTiles, true);
}

// Grid-wide "last CTA" detection: thread 0 fences (its tile partials become
// visible) and takes a ticket; true in every thread of the CTA that finished
// last among the kernel's gridDim.x CTAs.  Must be called by all threads.
// The ticket is one acq_rel atomic: release publishes the CTA's writes
// (ordered before it by the barrier, cumulatively), acquire makes every other
// CTA's released writes visible to the last one.  MPB_FENCED_TICKET=1 restores
// the fence / atomic / fence sequence.
__device__ __forceinline__ bool grid_last(unsigned int *ticket) {
  __shared__ int am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
#ifdef MPB_FENCED_TICKET
    __threadfence();
    am_last = atomicAdd(ticket, 1u) == gridDim.x - 1u;
    if (am_last) __threadfence();
#else
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
    am_last = old == gridDim.x - 1u;
#endif
  }
  __syncthreads();
  return am_last != 0;
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, 1-D) + mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// raise the expected transaction bytes of the current phase without arriving
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Off-critical-path wait (the producer waiting for a free stage): the thread
// is suspended in hardware instead of spinning, leaving issue slots to the
// consumer warps of the SM.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}
// global -> shared bulk copy; dst/src 16-B aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// global store with an L2 evict-first policy (data not read again soon)
__device__ __forceinline__ void st_evict_first(double *p, double v) {
#ifdef MPB_NO_EVICT_FIRST
  *p = v;
#else
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#endif
}
// global store with an L2 evict-last policy (a vector the next kernels
// gather; MPB_EVICT_LAST=1 enables it, else a plain store)
template <typename T>
__device__ __forceinline__ void st_keep(T *p, T v) {
#ifdef MPB_EVICT_LAST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (sizeof(T) == 8)
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(*reinterpret_cast<unsigned long long *>(&v)),
                 "l"(pol)
                 : "memory");
  else
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(*reinterpret_cast<unsigned *>(&v)), "l"(pol)
                 : "memory");
#else
  *p = v;
#endif
}
// The same for data read once per kernel (matrix values / columns): L2
// evict-first, so the streamed matrix does not push the iteration's vectors
// (gathered by the next kernels) out of L2.  MPB_NO_EVICT_FIRST=1: plain.
__device__ __forceinline__ void bulk_g2s_stream(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
#ifdef MPB_NO_EVICT_FIRST
  bulk_g2s(dst, src, bytes, bar);
#else
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#endif
}

// streaming loads (read once per kernel): L1 no-allocate, L2 evict-first
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float ld_stream(const float *p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor drains; everything before
// pdl_wait() must touch only data the predecessor does not write.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Staged byte window of elements [e0, e1) of an array: 16-B aligned outward.
// A 16-B granule never straddles a page, so the outward rounding never faults.
struct Window {
  uintptr_t g0;
  uint32_t bytes;
  uint32_t skew;  // byte offset of element e0 inside the window
};
template <typename E>
__device__ __forceinline__ Window window_of(const E *base, long long e0, long long e1) {
  uintptr_t a0 = reinterpret_cast<uintptr_t>(base + e0);
  uintptr_t a1 = reinterpret_cast<uintptr_t>(base + e1);
  Window w;
  w.g0 = a0 & ~uintptr_t(15);
  w.bytes = static_cast<uint32_t>(((a1 + 15) & ~uintptr_t(15)) - w.g0);
  w.skew = static_cast<uint32_t>(a0 - w.g0);
  return w;
}

// host+device: bytes of a staging region for cap_e elements of size es
__host__ __device__ constexpr uint32_t region_bytes(int cap_e, int es) {
  return ((static_cast<uint32_t>(cap_e) * es + 32 + 15) / 16) * 16;
}

template <typename T>
__device__ __forceinline__ T narrow_or_copy(double v);
template <>
__device__ __forceinline__ float narrow_or_copy<float>(double v) {
  return __double2float_rn(v);
}
template <>
__device__ __forceinline__ double narrow_or_copy<double>(double v) {
  return v;
}

// IEEE ops without contraction (belt and braces on top of --fmad=false)
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

}  // namespace mpb
