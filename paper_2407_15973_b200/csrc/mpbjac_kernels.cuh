// mpbjac_kernels.cuh — the sm_100a kernels of the mixed-precision BJAC-PCG
// hot path.
//
// Matrix layout: SELL-32 (sliced ELLPACK, slice height 32 = one warp, rows
// in original order).  Row r lives in slice r/32, lane r%32; its j-th stored
// entry (CSR order = ascending column) is at sp[r/32] + 32*j + r%32; padding
// slots carry column -1.  Every thread owns one row and accumulates it
// sequentially in ascending column order without FMA, which makes the kernels
// bit-identical to the reference's row-sequential numba kernels
// (pkg/src/mpcg/kernels_numba.py:37-70).
//
// Work unit: a tile of whole BJAC blocks (<= 256 rows), one thread per row.
// The hot kernels are persistent and warp-specialised: warp 8 of each CTA
// is a TMA producer that streams the inputs of the next tiles (SELL values,
// slice pointers, per-row metadata, the residual) into a ring of
// shared-memory stages (cp.async.bulk + full/empty mbarriers); warps 0-7 only
// compute.
//
// Column indices are not streamed.  Every row whose stored columns, taken as
// offsets from the row (c_j - row, in stored order), match one of <= 128
// "row patterns" of the matrix (a 7-point stencil has 27, a 3-T system 81)
// keeps only a pattern id in its 2-byte metadata, next to the slot range of
// its in-block entries: columns are rebuilt as row + offset from the pattern
// table held in shared memory.  Rows without a pattern ("generic" rows: long
// or irregular rows) read their SELL columns, staged only for tiles that
// contain such rows.  This removes 4 of the 8 bytes per fp32 entry (4 of 12
// per fp64 entry) of every pass.  Vector gathers (z_in, p) go through L1.
//
// Dot products follow the fixed tile-tree order of include/mpbjac_order.h.
// The scalar steps of the recurrence (rho, alpha, beta, relres, the aMP
// branch, error flags, trace) run in the last CTA of the kernel producing
// their partials, so an iteration is 4 kernels (k = 2).
#pragma once
#include <type_traits>

#include "mpbjac_device.cuh"

namespace mpb {

constexpr int kSlots = 9;                      // register-resident row entries (stencils, 3-T rows)
// Offset-slot ("DIA") layout of 7-point stencil plans: every row pattern's
// column offsets are a subset of the same kDiaSlots ascending offsets, so
// slot k of EVERY row is the entry at column row + doff[k] (absent entries:
// value 0 and a cleared bit in the row's presence mask).  Stored order =
// ascending column = ascending slot, so a row sum over the present slots is
// the same sequence of roundings as over the stored entries.
constexpr int kDiaSlots = 7;
constexpr int kDiaDiag = 3;                    // the diagonal's slot (offset 0)
#ifndef MPB_ROWS_PER_THREAD
#define MPB_ROWS_PER_THREAD 1
#endif
constexpr int kRowsPerThread = MPB_ROWS_PER_THREAD;  // tile rows per consumer thread
constexpr int kConsumers = kCtaThreads / kRowsPerThread;  // compute threads of the warp-specialised kernels
constexpr int kWsThreads = kConsumers + 32;    // + one TMA producer warp
// rows per consumer thread of the BJAC passes after the first (MPB_LAST_RPT=2:
// 4 consumer warps per CTA, 6 CTAs per SM; measured 0.8 % slower on C2 and
// 1.6 % on C4 than 1 row per thread, whose tails are shorter)
#ifndef MPB_LAST_RPT
#define MPB_LAST_RPT 1
#endif
constexpr int kLastRpt = MPB_LAST_RPT;
// final sums of the warp-specialised kernels: lanes per consumer thread
constexpr int kFinRptWs = kConsumers >= kFinThreads ? 1 : kFinThreads / kConsumers;
static_assert(kConsumers * kFinRptWs >= kFinThreads, "fin_sum lanes");
constexpr int kMaxStages = 4;
constexpr int kMaxPend = 4;  // owned chunks a producer keeps pending
// MPB_MINB_PASS / MPB_MINB_SPMV=n (experiments): compile the warp-specialised
// kernels for n co-resident CTAs per SM (caps their registers).  Unset: no
// minimum (not the same as 1 -- ptxas then picks the register budget itself)
#ifdef MPB_MINB_PASS
#define MPB_WS_BOUNDS_PASS __launch_bounds__(kWsThreads, MPB_MINB_PASS)
#else
#define MPB_WS_BOUNDS_PASS __launch_bounds__(kWsThreads)
#endif
// (SpMV: 4 CTAs per SM.  The two-level variant for 3-T rows took 72 registers / 3 CTAs on its
// own: C4's SpMV 139.5 -> 128.6 us with the cap, no spills; MPB_MINB_SPMV=0: no minimum)
#ifndef MPB_MINB_SPMV
#define MPB_MINB_SPMV 4
#endif
#if MPB_MINB_SPMV > 0
#define MPB_WS_BOUNDS_SPMV __launch_bounds__(kWsThreads, MPB_MINB_SPMV)
#else
#define MPB_WS_BOUNDS_SPMV __launch_bounds__(kWsThreads)
#endif
constexpr int kBarConsumers = 1;               // named barrier id among consumers
// full-tile fast path of the passes after the first (bjac_tile_full); MPB_FAST=0 compiles it out
#ifndef MPB_FAST
#define MPB_FAST 1
#endif
constexpr bool kFastTiles = MPB_FAST != 0;
constexpr uint16_t kMetaGeneric = 0xFFFFu;

// ---- row patterns ------------------------------------------------------------
constexpr int kPatMax = 128;     // pattern ids 0..127
constexpr int kPatStride = 10;   // ints per table entry: len | dpos << 8, then kSlots offsets
constexpr int kPatHash = 4096;   // slots of the setup-time pattern hash table (power of 2)
constexpr uint8_t kPidGeneric = 255;
struct PatSlot {
  unsigned long long key;  // 0 = empty
  int count, rep;          // rows with the pattern, one of them
};

// ---- per-row metadata: pid | i0 << 8 | i1 << 12, or kMetaGeneric -------------
// (pid < kPatMax, so a pattern row never reads as kMetaGeneric)
__device__ __forceinline__ int meta_pid(uint16_t m) { return m & 0xFF; }
__device__ __forceinline__ int meta_i0(uint16_t m) { return (m >> 8) & 15; }
__device__ __forceinline__ int meta_i1(uint16_t m) { return m >> 12; }
__device__ __forceinline__ int pat_len(int hdr) { return hdr & 0xFF; }
__device__ __forceinline__ int pat_dpos(int hdr) { return hdr >> 8; }

// the pattern table into shared memory (all threads of the CTA, before the
// __syncthreads of ring_init)
__device__ __forceinline__ void load_patterns(int *s_pat, const int *pat, int npat) {
  for (int i = threadIdx.x; i < npat * kPatStride; i += blockDim.x) s_pat[i] = __ldg(pat + i);
}

// ---------------------------------------------------------------------------
// scalar steps of the recurrence (solver.py:128-177, policies.py:102-116)
// ---------------------------------------------------------------------------
// kStepRrZ: kStepRr after the fused update, which also ran the next
// iteration's first BJAC pass for the current branch (valid iff it stays)
enum ScalarStep {
  kStepR0 = 0, kStepRho = 1, kStepPq = 2, kStepRr = 3, kStepTrue = 4, kStepFinal = 5, kStepStart = 6, kStepRrZ = 7
};

__device__ __forceinline__ int choose_branch(int kind, double tol, double relres) {
  if (kind == 0) return 0;
  if (kind == 1) return 1;
  if (kind == 2) return relres >= tol ? 0 : 1;
  return relres >= tol ? 1 : 0;
}

// the solve graph's device-side loop continues while the solve is not done.
// The while condition is 1 from the graph launch on (cudaGraphCondAssignDefault)
// and only ever needs clearing: cudaGraphSetConditional delays the grid's
// completion by ~2.5 us, so it is called once, when the solve is done.
__device__ __forceinline__ void set_loop(const SolverState *st) {
  if (st->cond != 0ull && st->done) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(st->cond), 0u);
}

__device__ __forceinline__ void fail(SolverState *st, int code, double val) {
  st->error = code;
  st->err_it = st->it;
  st->err_val = val;
  st->done = 1;
  set_loop(st);
}

// Executed by one thread once the global sum `tot` of a step is known.
// Inlined where the step is a constant (the switch folds), on a state copy
// in shared memory (finish_grid) or registers.
// trace: false skips the trace-array writes (k_solve_small: every CTA runs
// the steps on its own state copy, CTA 0 alone writes the trace)
__device__ __forceinline__ void scalar_step_body(int step, double tot, SolverState *st, bool trace = true) {
  switch (step) {
    case kStepR0: {
      st->r0 = sqrt(tot);
      st->relres = 1.0;
      st->it = 1;
      st->first = 1;
      st->branch = choose_branch(st->kind, st->adp_tol, 1.0);
      if (st->r0 == 0.0) {
        st->converged = 1;
        st->done = 1;
      }
      break;
    }
    case kStepRho: {
      tl_mark(st, 0, 2, true);
      if (st->ovf_count != 0ull) {
        fail(st, kNarrowOverflow, 0.0);
        break;
      }
      st->rho = tot;
      if (tot == 0.0) { fail(st, kBreakdown, tot); break; }
      if (tot < 0.0) { fail(st, kIndefPrecond, tot); break; }
      st->beta = st->first ? 0.0 : tot / st->rho_prev;
      break;
    }
    case kStepPq: {
      tl_mark(st, 1, 2, true);
      st->pq = tot;
      if (tot <= 0.0) { fail(st, kIndefMatrix, tot); break; }
      st->alpha = st->rho / tot;
      st->upd_branch = st->branch;
      break;
    }
    case kStepRr:
    case kStepRrZ: {
      tl_mark(st, 2, 2, true);
      const int old_branch = st->branch;
      const double rnorm = sqrt(tot);
      st->rnorm = rnorm;
      st->rho_prev = st->rho;
      st->first = 0;
      if (!isfinite(rnorm)) { fail(st, kNonFinite, rnorm); break; }
      const double relres = rnorm / st->r0;
      st->relres = relres;
      const long long it = st->it;
      if (trace) {
        st->tr_relres[it - 1] = relres;
        st->tr_branch[it - 1] = st->branch;
        st->tr_time[it - 1] = 1e-9 * static_cast<double>(globaltimer_ns() - st->t0_ns);
      }
      st->last_it = it;
      st->true_pending = (st->stride > 0 && it % st->stride == 0) ? 1 : 0;
      if (relres <= st->res_tol) {
        st->converged = 1;
        st->done = 1;
      } else if (it >= st->cap) {
        st->done = 1;
      } else {
        st->it = it + 1;
        st->branch = choose_branch(st->kind, st->adp_tol, relres);
      }
      st->z1_ok = (step == kStepRrZ && st->branch == old_branch) ? 1 : 0;
      if (step == kStepRrZ && st->branch != old_branch) {  // speculative narrowing no longer applies
        st->ovf_count = 0ull;
        st->ovf_first = 0x7fffffffffffffffLL;
      }
      set_loop(st);
      break;
    }
    case kStepTrue: {
      st->tr_true[st->last_it - 1] = sqrt(tot) / st->r0;
      st->true_pending = 0;
      break;
    }
    case kStepFinal: {
      const double v = sqrt(tot) / st->r0;
      st->final_true = v;
      if (st->converged && st->last_it > 0 && isnan(st->tr_true[st->last_it - 1])) st->tr_true[st->last_it - 1] = v;
      break;
    }
    case kStepStart: {
      st->t0_ns = globaltimer_ns();
      break;
    }
  }
}

__device__ __noinline__ void scalar_step(int step, double tot, SolverState *st) { scalar_step_body(step, tot, st); }

// The scalar steps run on a register/local copy of the state: one batch of
// independent loads instead of a chain of dependent global round trips (the
// step sits on the critical path between two kernels).  state_store writes
// back what a step may change: the scalars (rho .. ovf_first) and the flags
// (dist .. pad) -- not the trace pointers, tickets, all-reduce buffers, loop
// handle or diagnostics pointer.
constexpr int kStWords = static_cast<int>(sizeof(SolverState) / 8);
static_assert(sizeof(SolverState) % 8 == 0, "state words");
static_assert(offsetof(SolverState, tr_relres) % 8 == 0 && offsetof(SolverState, dist) % 8 == 0 &&
                  offsetof(SolverState, cond) % 8 == 0,
              "state write-back ranges");
__device__ __forceinline__ void state_store(SolverState *g, const SolverState &L) {
  const unsigned long long *s = reinterpret_cast<const unsigned long long *>(&L);
  unsigned long long *d = reinterpret_cast<unsigned long long *>(g);
#pragma unroll
  for (int i = 0; i < static_cast<int>(offsetof(SolverState, tr_relres) / 8); i++) d[i] = s[i];
#pragma unroll
  for (int i = static_cast<int>(offsetof(SolverState, dist) / 8); i < static_cast<int>(offsetof(SolverState, cond) / 8);
       i++)
    d[i] = s[i];
}
__device__ __forceinline__ void state_load(SolverState &L, const SolverState *g) {
  const unsigned long long *s = reinterpret_cast<const unsigned long long *>(g);
  unsigned long long *d = reinterpret_cast<unsigned long long *>(&L);
#pragma unroll
  for (int i = 0; i < kStWords; i++) d[i] = __ldcg(s + i);
}

// After a kernel's CTAs have written all tile partials: the CTA that
// finishes last reduces them in the fixed order and runs the scalar step.
// The state is fetched into shared memory while the partials are summed.
// Called by all threads of the CTA.
// The chunk sums of the two-level order are in ck.csum: their owners stored
// them before their CTAs took the ticket (chunks_in_cta: the last CTA sums
// them here).
// One-level order (!ck.poll): the final CTA sums all tile partials.  Two
// levels: the chunk sums are in ck.csum, stored by their owners before their
// CTAs took the ticket (in_cta: grids that may exceed residency have no
// owners; the final CTA sums the chunks here).
template <int B = 16, int RPT = 1>
__device__ __forceinline__ void finish_grid(SolverState *st, int ticket, int step, const ChunkCtx &ck, double *ws,
                                            bool in_cta = false) {
  if (st == nullptr) return;
  if (!grid_last(&st->ticket[ticket])) return;
  __shared__ __align__(16) unsigned long long s_state[kStWords];
  if (threadIdx.x < kStWords) s_state[threadIdx.x] = __ldcg(reinterpret_cast<const unsigned long long *>(st) + threadIdx.x);
  if (ck.poll && in_cta) chunk_all_in_cta(ck);
  if (threadIdx.x == 0) tl_mark(st, step == kStepRho ? 0 : (step == kStepPq ? 1 : 2), 3, true);  // diagnostics
  const int nch = (ck.ntiles + kChunkTiles - 1) / kChunkTiles;
  const double tot = ck.poll ? fin_sum<B, RPT>(ck.csum, nch, ws)
                             : fin_sum<B, RPT>(ck.part, ck.ntiles, ws);  // (their barriers publish s_state)
  SolverState *L = reinterpret_cast<SolverState *>(s_state);
  const bool dist = L->dist != 0;
  if (threadIdx.x == 0) {
    if (dist) {  // multi-GPU: all-reduce first, k_apply_step runs the step
      st->red_local[0] = tot;
      st->red_local[1] = static_cast<double>(L->ovf_count);
    } else {
      scalar_step_body(step, tot, L);
    }
    st->ticket[ticket] = 0u;
  }
  if (!dist && threadIdx.x < 32) {  // warp 0 writes the changed state back (state_store's ranges)
    __syncwarp();
    unsigned long long *d = reinterpret_cast<unsigned long long *>(st);
    constexpr int a1 = static_cast<int>(offsetof(SolverState, tr_relres) / 8);
    constexpr int b0 = static_cast<int>(offsetof(SolverState, dist) / 8), b1 = static_cast<int>(offsetof(SolverState, cond) / 8);
    for (int i = threadIdx.x; i < a1 + (b1 - b0); i += 32) {
      const int w = i < a1 ? i : b0 + (i - a1);
      d[w] = s_state[w];
    }
  }
}

// One-level sums, streamed: instead of the kernel's last CTA summing every
// tile partial after the last tile (C2: 8,192 partials, 2-4 us on the
// critical path between two kernels, after a grid ticket), ONE warp of the
// grid (CTA 0, which takes no tiles) carries the 256 lane sums of the
// one-level order while the kernel runs: row c of the partials (tiles
// 256 c .. 256 c + 255) completes roughly in order of c; the warp polls the
// rows in order (each slot its own completion flag, kPartEmpty), lane l adding
// slots l, l + 32, .. of each row to its 8 lane sums -- lane j of 256 still
// adds partials j, j + 256, .. in ascending order from +0 -- and empties
// them.  After the last row: the 256-lane tree (8 virtual warps' butterflies,
// then the butterfly of their sums) and the scalar step, one L2 round trip
// after the last tile's partial lands.  Same additions in the same order as
// fin_sum: bit-identical.  The state snapshot is taken once at the start
// (only this step changes it during the kernel).  Called by one warp.
__device__ __forceinline__ void reduce_stream(SolverState *st, int step, double *part, int ntiles) {
  __shared__ __align__(16) unsigned long long s_rstate[kStWords];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kStWords; i += 32) s_rstate[i] = __ldcg(reinterpret_cast<const unsigned long long *>(st) + i);
  constexpr int W = kChunkTiles / 32;
  double acc[W];
#pragma unroll
  for (int w = 0; w < W; w++) acc[w] = 0.0;
  const int nrows = (ntiles + kChunkTiles - 1) / kChunkTiles;
  for (int c = 0; c < nrows;) {
    unsigned long long b0[W], b1[W];
    const bool two = c + 1 < nrows;
    bool f0 = true, f1 = true;
#pragma unroll
    for (int w = 0; w < W; w++) {
      const int i0 = c * kChunkTiles + 32 * w + lane, i1 = i0 + kChunkTiles;
      b0[w] = i0 < ntiles ? get_part_bits(part + i0) : 0ull;
      b1[w] = (two && i1 < ntiles) ? get_part_bits(part + i1) : 0ull;
      f0 = f0 && b0[w] != kPartEmpty;
      f1 = f1 && b1[w] != kPartEmpty;
    }
    f0 = __all_sync(0xffffffffu, f0);
    f1 = __all_sync(0xffffffffu, f1) && f0 && two;
    if (!f0) continue;
#pragma unroll
    for (int w = 0; w < W; w++) {
      const int i0 = c * kChunkTiles + 32 * w + lane;
      if (i0 < ntiles) {
        acc[w] = __dadd_rn(acc[w], __longlong_as_double(static_cast<long long>(b0[w])));
        reinterpret_cast<unsigned long long *>(part)[i0] = kPartEmpty;
      }
    }
    c++;
    if (f1) {
#pragma unroll
      for (int w = 0; w < W; w++) {
        const int i1 = c * kChunkTiles + 32 * w + lane;
        if (i1 < ntiles) {
          acc[w] = __dadd_rn(acc[w], __longlong_as_double(static_cast<long long>(b1[w])));
          reinterpret_cast<unsigned long long *>(part)[i1] = kPartEmpty;
        }
      }
      c++;
    }
  }
  // block_tree<256>: virtual warp w = slots 32 w + lane
  double r = 0.0;
#pragma unroll
  for (int w = 0; w < W; w++) {
    const double v = warp_bfly(acc[w]);
    if (lane == w) r = v;
  }
  const double tot = warp_bfly(r);
  SolverState *L = reinterpret_cast<SolverState *>(s_rstate);
  __syncwarp();
  const bool dist = L->dist != 0;
  if (lane == 0) {
    if (dist) {  // multi-GPU: all-reduce first, k_apply_step runs the step
      st->red_local[0] = tot;
      st->red_local[1] = static_cast<double>(L->ovf_count);
    } else {
      scalar_step_body(step, tot, L);
    }
  }
  __syncwarp();
  if (!dist) {  // the changed state words (state_store's ranges)
    unsigned long long *d = reinterpret_cast<unsigned long long *>(st);
    constexpr int a1 = static_cast<int>(offsetof(SolverState, tr_relres) / 8);
    constexpr int b0 = static_cast<int>(offsetof(SolverState, dist) / 8), b1 = static_cast<int>(offsetof(SolverState, cond) / 8);
    for (int i = lane; i < a1 + (b1 - b0); i += 32) {
      const int wd = i < a1 ? i : b0 + (i - a1);
      d[wd] = s_rstate[wd];
    }
  }
}

// in-process slab group: red_global of every rank = the ranks' red_local
// summed in rank order (for two ranks the same value as NCCL's sum)
constexpr int kMaxLocalRanks = 16;
struct LocalStates {
  SolverState *p[kMaxLocalRanks];
};
__global__ void k_local_allreduce(LocalStates sts, int nranks) {
  if (threadIdx.x > 1) return;
  const int i = threadIdx.x;
  double acc = sts.p[0]->red_local[i];
  for (int r = 1; r < nranks; r++) acc = __dadd_rn(acc, sts.p[r]->red_local[i]);
  for (int r = 0; r < nranks; r++) sts.p[r]->red_global[i] = acc;
}

// multi-GPU: the scalar step on the all-reduced sum (every rank computes the
// same state from the same global values)
__global__ void k_apply_step(int step, SolverState *st, int gate) {
  if (threadIdx.x != 0) return;
  SolverState L;
  state_load(L, st);
  if (gate == 1 && !L.true_pending) return;
  if (gate == 2 && L.done) return;
  if (step == kStepRho) L.ovf_count = static_cast<unsigned long long>(L.red_global[1]);
  scalar_step(step, L.red_global[0], &L);
  state_store(st, L);
}

// U independent tile sums at once (same order as block_tree<kTileThreads>
// for each): one pair of barriers for all U.  Result u valid in thread 0.
template <int U>
__device__ __forceinline__ void block_tree_multi(double (&v)[U], double (*ws)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < U; u++) v[u] = warp_bfly(v[u]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < U; u++) ws[u][warp] = v[u];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const double r = lane < kTileThreads / 32 ? ws[u][lane] : 0.0;
      v[u] = warp_bfly(r);
    }
  }
}

// ---------------------------------------------------------------------------
// tiles: descriptor, geometry, TMA stage layout
// ---------------------------------------------------------------------------
struct TileDesc {
  int lo, hi;   // rows [lo, hi)
  int s0, s1;   // SELL slices [s0, s1)
  int e0, e1;   // SELL entries [e0, e1) = [sp[s0], sp[s1]) (multiples of 32)
  int bf, nbk;  // blocks bf .. bf+nbk-1 overlap the tile
  int ie0, ie1; // in-block SELL entries [ib_sp[s0], ib_sp[s1])
  int ngen;     // generic rows (kMetaGeneric) in the tile
  int pad1;
};

struct TileGeom {
  int ntiles;
  int poll;    // two-level sums: chunk owners poll (ChunkCtx::poll)
  int cap_e;   // staged SELL entries per tile (max over tiles, capped)
  int max_sl;  // max slices per tile
  int ns;      // shared-memory stages (prefetch depth)
  int cols;    // stages carry a column region (the plan has generic rows)
  int npat;    // row patterns in the table
  int kib;     // most in-block entries of a row
  int ub;      // every block has this many rows (0: blocks differ)
  int red;     // one-level sums streamed by CTA 0's first warp (reduce_stream); CTA 0 takes no tiles
};

// Byte offsets of one shared-memory stage.
struct StageLayout {
  uint32_t col, val, sp, meta, v0, v1, v2, v3, bytes;
  uint32_t win;  // start of the gather windows (bjac_layout with windows), else == bytes
};
__host__ __device__ constexpr uint32_t al16u(uint32_t b) { return (b + 15u) & ~15u; }
// v*es: element sizes of up to three row-vector slices [lo, hi) (0: absent)
__host__ __device__ inline StageLayout stage_layout(int cap_e, int es, int max_sl, bool cols, bool meta, int v0es,
                                                    int v1es, int v2es, int v3es = 0) {
  StageLayout L;
  uint32_t off = 0;
  L.col = off;
  off += cols ? al16u(static_cast<uint32_t>(cap_e) * 4u) : 0u;
  L.val = off;
  off += al16u(static_cast<uint32_t>(cap_e) * es);
  L.sp = off;
  off += al16u(static_cast<uint32_t>(max_sl + 1) * 4u + 16u);
  L.meta = off;
  off += meta ? al16u(static_cast<uint32_t>(kTileRows) * 2u + 16u) : 0u;
  L.v0 = off;
  off += v0es ? al16u(static_cast<uint32_t>(kTileRows) * v0es + 16u) : 0u;
  L.v1 = off;
  off += v1es ? al16u(static_cast<uint32_t>(kTileRows) * v1es + 16u) : 0u;
  L.v2 = off;
  off += v2es ? al16u(static_cast<uint32_t>(kTileRows) * v2es + 16u) : 0u;
  L.v3 = off;
  off += v3es ? al16u(static_cast<uint32_t>(kTileRows) * v3es + 16u) : 0u;
  L.bytes = off;
  L.win = off;
  return L;
}

// ---- z_in gather windows (passes after the first) --------------------------
// The plan's row patterns use few distinct column offsets (a 7-point stencil:
// -n^2, -n, -1, 0, 1, n, n^2), clustered into <= kMaxWin intervals [a, b].
// A stage then also holds z_in rows [lo + a, hi + b) of each window, copied
// with TMA, so the pass gathers z_in from shared memory instead of global
// loads.  Window k's region starts at win_off(k) after the stage's other
// data; global row g sits at byte  (g - lo) es - floor16(a es)  of it (tiles
// start at a multiple of 4 rows, so the skew is the same for every tile).
constexpr int kMaxWin = 6;
constexpr int kWinMaxRows = 2048;
struct WinSet {
  int n;              // windows (0: gather from global memory)
  int zlen;           // rows of z_in (multi-GPU slabs: own rows + ghosts)
  int a[kMaxWin], b[kMaxWin];
};
__host__ __device__ inline int floor16i(int x) { return x & ~15; }
__host__ __device__ inline uint32_t win_region_bytes(const WinSet &w, int k, int es) {
  return al16u(static_cast<uint32_t>((kTileRows + w.b[k] - w.a[k]) * es + 32));
}
__host__ __device__ inline uint32_t win_off(const WinSet &w, int k, int es) {
  uint32_t off = 0;
  for (int j = 0; j < k; j++) off += win_region_bytes(w, j, es);
  return off;
}

// Ring of shared-memory stages filled by the producer warp.
template <int MS>
struct RingT {
  uint64_t full[MS];   // TMA bytes landed
  uint64_t empty[MS];  // consumers done with the stage
  int ok[MS];          // tile fitted and was staged
  int tile[MS];        // tile in the stage, -1: no more tiles
  TileDesc desc[MS];
  int pend[kMaxPend];  // producer: owned chunks not yet summed
};
using Ring = RingT<kMaxStages>;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename E>
__device__ __forceinline__ void tma_window(unsigned char *dst, const E *base, int lo, int hi, uint64_t *bar,
                                           bool last_use = false) {
  const Window w = window_of(base, lo, hi);
  if (last_use) bulk_g2s_stream(dst, reinterpret_cast<const void *>(w.g0), w.bytes, bar);
  else bulk_g2s(dst, reinterpret_cast<const void *>(w.g0), w.bytes, bar);
}
template <typename E>
__device__ __forceinline__ uint32_t window_bytes(const E *base, int lo, int hi) {
  return base == nullptr ? 0u : window_of(base, lo, hi).bytes;
}
template <typename E>
__device__ __forceinline__ const E *staged(const unsigned char *region, const E *base, int lo, int hi) {
  return reinterpret_cast<const E *>(region + window_of(base, lo, hi).skew);
}

// Producer: stage tile `tile` into ring slot st (thread = producer lane 0).
// part: kFillAll, or kFillStatic (the matrix data: columns, values, slice
// pointers, row metadata -- no arrive, so it may run before the grid
// dependency wait) followed later by kFillDynamic (the vector slices + the
// arrive that completes the stage).
enum { kFillAll = 0, kFillStatic = 1, kFillDynamic = 2 };

// LAST_USE: bit i set = vector slice vi is read for the last time this
// iteration (streamed evict-first, like the matrix data)
// win / zwin (passes after the first): the z_in gather windows of the tile,
// dynamic data like the vector slices (the previous pass wrote z_in).
template <typename T, typename V0, typename V1, typename V2, bool IB = false, typename V3 = uint8_t,
          unsigned LAST_USE = 0u, class RG>
__device__ __forceinline__ void produce(RG &R, int st, const TileDesc *td, int tile, const TileGeom &g,
                                        const StageLayout &L, unsigned char *stage, const int *sp, const int *scol,
                                        const T *sval, const uint16_t *meta, const V0 *v0, const V1 *v1,
                                        const V2 *v2, const V3 *v3 = nullptr, int part = kFillAll,
                                        const WinSet *win = nullptr, const T *zwin = nullptr) {
  TileDesc d;
  if (part != kFillDynamic) {
    d = td[tile];
    R.desc[st] = d;
  } else {
    d = R.desc[st];
  }
  const int e0 = IB ? d.ie0 : d.e0, e1 = IB ? d.ie1 : d.e1;
  const int nent = e1 - e0;
  const bool fits = nent <= g.cap_e && (d.s1 - d.s0) <= g.max_sl;
  if (part != kFillDynamic) {
    R.ok[st] = fits ? 1 : 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (!fits) {
    if (part != kFillStatic) mbar_arrive(&R.full[st]);
    return;
  }
  const bool cols = g.cols && d.ngen > 0;  // pattern rows rebuild their columns
  const uint32_t sbytes = static_cast<uint32_t>(nent) * ((cols ? 4u : 0u) + sizeof(T)) +
                          window_bytes(sp, d.s0, d.s1 + 1) + window_bytes(meta, d.lo, d.hi);
  uint32_t dbytes = window_bytes(v0, d.lo, d.hi) + window_bytes(v1, d.lo, d.hi) + window_bytes(v2, d.lo, d.hi) +
                    window_bytes(v3, d.lo, d.hi);
  // gather window k: z_in rows [lo + a_k, hi + b_k) clamped to [0, zlen); its
  // element g lands at byte (g - lo) es - floor16(a_k es) of the window region
  constexpr int es = sizeof(T);
  const int nwin = win != nullptr ? win->n : 0;
  for (int k = 0; k < nwin; k++) {
    const int gs = max(d.lo + win->a[k], 0), ge = min(d.hi + win->b[k], win->zlen);
    if (gs < ge) dbytes += static_cast<uint32_t>(((ge * es + 15) & ~15) - floor16i(gs * es));
  }
  if (part == kFillAll) mbar_arrive_expect_tx(&R.full[st], sbytes + dbytes);
  if (part == kFillStatic) mbar_expect_tx(&R.full[st], sbytes);
  if (part != kFillDynamic) {
    if (cols) bulk_g2s_stream(stage + L.col, scol + e0, static_cast<uint32_t>(nent) * 4u, &R.full[st]);
    bulk_g2s_stream(stage + L.val, sval + e0, static_cast<uint32_t>(nent) * sizeof(T), &R.full[st]);
    tma_window(stage + L.sp, sp, d.s0, d.s1 + 1, &R.full[st]);
    if (meta != nullptr) tma_window(stage + L.meta, meta, d.lo, d.hi, &R.full[st]);
  }
  if (part == kFillStatic) return;
  if (part == kFillDynamic) mbar_arrive_expect_tx(&R.full[st], dbytes);
  if (v0 != nullptr) tma_window(stage + L.v0, v0, d.lo, d.hi, &R.full[st], LAST_USE & 1u);
  if (v1 != nullptr) tma_window(stage + L.v1, v1, d.lo, d.hi, &R.full[st], LAST_USE & 2u);
  if (v2 != nullptr) tma_window(stage + L.v2, v2, d.lo, d.hi, &R.full[st], LAST_USE & 4u);
  if (v3 != nullptr) tma_window(stage + L.v3, v3, d.lo, d.hi, &R.full[st], LAST_USE & 8u);
  uint32_t woff = L.win;
  for (int k = 0; k < nwin; k++) {
    const int gs = max(d.lo + win->a[k], 0), ge = min(d.hi + win->b[k], win->zlen);
    if (gs < ge) {
      const int src0 = floor16i(gs * es), g0 = d.lo * es + floor16i(win->a[k] * es);
      bulk_g2s(stage + woff + (src0 - g0), reinterpret_cast<const unsigned char *>(zwin) + src0,
               static_cast<uint32_t>(((ge * es + 15) & ~15) - src0), &R.full[st]);
    }
    woff += win_region_bytes(*win, k, es);
  }
}

// Producer loop (producer warp, lane 0): claims tiles from the launch's
// counter (dynamic scheduling: CTAs that start late or run slow take fewer
// tiles), waiting for a stage to be released before refilling it, and ends
// the consumers' walk with tile -1.  The globally last claim (ntiles +
// gridDim claims in all) resets the counter for the next launch.  ctr ==
// null: static walk blockIdx.x, +gridDim.x, ...
//
// prefetch (fixed-branch solves): the matrix data of the first ns tiles is
// requested before the grid dependency wait -- it does not depend on the
// previous kernel -- so it streams while the previous kernel drains; the
// vector slices follow after the wait.  gated() is evaluated after the wait;
// a gated-off launch drains its prefetched copies and stops (the solve
// resets the claim counters at its start and end).
//
// The whole producer warp runs the loop (lane 0 claims and issues the
// copies).  Chunk duties (ck.csum != null): claiming the last tile of a
// chunk makes this warp the chunk's owner (chunk_poll).  Pending chunks are
// polled while the producer would otherwise wait for a stage to come back,
// and blocking after the last claim.  (Owners polling from a consumer warp
// stall their CTA: measured slower.)
// L1 prefetch of a tile descriptor (48 bytes, may straddle two lines)
__device__ __forceinline__ void prefetch_desc(const TileDesc *td, int tile) {
  if (td == nullptr || tile < 0) return;
  const char *p = reinterpret_cast<const char *>(td + tile);
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + sizeof(TileDesc) - 1));
}

// End markers (one thread): stage st (free) and the next nterm - 1 stages
// get tile -1, so that each of nterm consumer warps sees one (warp-per-tile
// kernels consume the stages round-robin, stage i by warp i % nterm).
template <class RG>
__device__ __forceinline__ void ring_end(RG &R, int st, int rnd, int ns, int nterm) {
  R.tile[st] = -1;
  mbar_arrive(&R.full[st]);
  for (int i = 1; i < nterm; i++) {
    if (++st == ns) {
      st = 0;
      rnd++;
    }
    if (rnd > 0) mbar_wait_sleep(&R.empty[st], (rnd - 1) & 1);
    R.tile[st] = -1;
    mbar_arrive(&R.full[st]);
  }
}

template <typename F, typename G, class RG>
__device__ __forceinline__ void producer_loop(RG &R, int ntiles, int ns, unsigned int *ctr, bool prefetch,
                                              G &&gated, F &&fill, const ChunkCtx &ck, int nterm = 1,
                                              const TileDesc *td = nullptr) {
  const int lane = threadIdx.x & 31;
  int next = blockIdx.x;
  auto claim = [&]() -> int {
    int t = -1;
    if (lane == 0) {
      if (ctr != nullptr) {
        const unsigned int v = atomicAdd(ctr, 1u);
        if (v == static_cast<unsigned int>(ntiles) + gridDim.x - 1u) atomicExch(ctr, 0u);
        t = v < static_cast<unsigned int>(ntiles) ? static_cast<int>(v) : -1;
      } else {
        t = next < ntiles ? next : -1;
      }
    }
    next += gridDim.x;
    return __shfl_sync(0xffffffffu, t, 0);
  };
  // owned chunks not yet summed: a FIFO in shared memory, [phead, ptail)
  int phead = 0, ptail = 0;
  auto own = [&](int tile) {
    if (ck.csum == nullptr || !chunk_final(tile, ntiles)) return;
    if (ptail - phead == kMaxPend) chunk_poll(ck, R.pend[phead++ % kMaxPend], true);
    if (lane == 0) R.pend[ptail % kMaxPend] = tile / kChunkTiles;
    __syncwarp();
    ptail++;
  };
  auto poll_oldest = [&](bool block) {
    if (phead != ptail && chunk_poll(ck, R.pend[phead % kMaxPend], block)) phead++;
  };
  int npre = 0;
  bool exhausted = false;
  if (prefetch) {
    for (; npre < ns; npre++) {
      const int tile = claim();
      if (lane == 0) R.tile[npre] = tile;
      if (tile < 0) {
        exhausted = true;
        break;
      }
      if (lane == 0) fill(npre, tile, kFillStatic);
      own(tile);
    }
  }
  pdl_wait();
  if (gated()) {
    if (lane == 0) {
      for (int i = 0; i < npre; i++) {  // let the copies land before the CTA exits
        mbar_arrive(&R.full[i]);
        mbar_wait(&R.full[i], 0);
      }
    }
    __syncwarp();
    return;
  }
  if (lane == 0)
    for (int i = 0; i < npre; i++) fill(i, R.tile[i], kFillDynamic);
  int st = npre % ns, rnd = npre / ns;  // stage, and how often it has been filled before
  if (!exhausted) {
    // one claim ahead: the next tile is claimed (and its descriptor
    // prefetched) after the current stage's copies are issued, so neither
    // round trip sits between a free stage and its refill
    int cur = claim();
    if (lane == 0) prefetch_desc(td, cur);
    for (;;) {
      if (rnd > 0) {
        if (phead != ptail && !mbar_test(&R.empty[st], (rnd - 1) & 1)) poll_oldest(false);
        mbar_wait_sleep(&R.empty[st], (rnd - 1) & 1);
      }
      const int tile = cur;
      if (lane == 0) R.tile[st] = tile;
      if (tile < 0) break;
      if (lane == 0) fill(st, tile, kFillAll);
      own(tile);
      cur = claim();
      if (lane == 0) prefetch_desc(td, cur);
      if (++st == ns) {
        st = 0;
        rnd++;
      }
    }
  }
  if (lane == 0) ring_end(R, st, rnd, ns, nterm);  // stage st holds the (first) end marker
  __syncwarp();
  while (phead != ptail) poll_oldest(true);
}

// Single-lane producer (lane 0 of the producer warp) for kernels without
// chunk owners: the same walk as producer_loop.
// nclaim: CTAs that claim tiles (each makes exactly one failing claim; 0: the whole grid)
template <typename F, typename G, class RG>
__device__ __forceinline__ void producer_loop_single(RG &R, int ntiles, int ns, unsigned int *ctr, bool prefetch,
                                              G &&gated, F &&fill, int nterm = 1, const TileDesc *td = nullptr,
                                              unsigned int nclaim = 0u) {
  int next = blockIdx.x;
  if (nclaim == 0u) nclaim = gridDim.x;
  auto claim = [&]() -> int {
    if (ctr != nullptr) {
      const unsigned int v = atomicAdd(ctr, 1u);
      if (v == static_cast<unsigned int>(ntiles) + nclaim - 1u) atomicExch(ctr, 0u);
      return v < static_cast<unsigned int>(ntiles) ? static_cast<int>(v) : -1;
    }
    const int t = next < ntiles ? next : -1;
    next += gridDim.x;
    return t;
  };
  int npre = 0;
  bool exhausted = false;
  if (prefetch) {
    for (; npre < ns; npre++) {
      const int tile = claim();
      R.tile[npre] = tile;
      if (tile < 0) {
        exhausted = true;
        break;
      }
      fill(npre, tile, kFillStatic);
    }
  }
  pdl_wait();
  if (gated()) {
    for (int i = 0; i < npre; i++) {  // let the copies land before the CTA exits
      mbar_arrive(&R.full[i]);
      mbar_wait(&R.full[i], 0);
    }
    return;
  }
  for (int i = 0; i < npre; i++) fill(i, R.tile[i], kFillDynamic);
  if (exhausted) {
    ring_end(R, npre, 0, ns, nterm);
    return;
  }
  int st = npre % ns, rnd = npre / ns;  // stage, and how often it has been filled before
  int cur = claim();  // one claim ahead (producer_loop)
  prefetch_desc(td, cur);
  for (;;) {
    if (rnd > 0) mbar_wait_sleep(&R.empty[st], (rnd - 1) & 1);
    const int tile = cur;
    R.tile[st] = tile;
    if (tile < 0) {
      ring_end(R, st, rnd, ns, nterm);
      return;
    }
    fill(st, tile, kFillAll);
    cur = claim();
    prefetch_desc(td, cur);
    if (++st == ns) {
      st = 0;
      rnd++;
    }
  }
}

// consumer-side ring cursor: stage and mbarrier parity of the i-th tile
struct RingCursor {
  int st = 0, phase = 0;
  __device__ __forceinline__ void advance(int ns) {
    if (++st == ns) {
      st = 0;
      phase ^= 1;
    }
  }
};

template <class RG>
__device__ __forceinline__ void ring_init(RG &R, int ns, int consumers = kConsumers) {
  if (threadIdx.x == 0) {
    for (int st = 0; st < ns; st++) {
      mbar_init(&R.full[st], 1);
      mbar_init(&R.empty[st], consumers / 32);
    }
  }
  __syncthreads();
}

// consumer warp releases its use of a stage (one arrive per warp)
template <class RG>
__device__ __forceinline__ void ring_release(RG &R, int st) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&R.empty[st]);
}

// ---------------------------------------------------------------------------
// fused block-Jacobi pass: z_out = z_in + D_b^{-1}(r - A z_in)
// (bjac.py:127-149 one outer pass; kernels_numba.py:48-70 the t inner sweeps)
// ---------------------------------------------------------------------------
template <typename T>
struct PassArgs {
  const int *sp;         // SELL slice_ptr
  const int *scol;       // SELL columns (-1 = padding; generic rows only)
  const T *sval;         // SELL values in storage precision
  const int *ib_sp;      // in-block SELL (first pass): slice_ptr
  const int *ib_col;     //   columns (generic rows only)
  const T *ib_val;       //   values
  const uint16_t *meta;  // per-row static structure (plan-bound)
  const int *pat;        // row-pattern table (g.npat entries of kPatStride ints)
  const TileDesc *td;    // tile descriptors
  unsigned int *ctr;     // tile-claim counter of the launch (null: static walk)
  const int *boff;       // nb+1 block offsets (generic rows, large blocks)
  TileGeom g;
  int t;
  const double *r64;     // fp64 residual, narrowed on load for T=float ...
  const T *rT;           // ... or a residual already in T (when r64 == null)
  const T *zin;          // previous pass output (null on the first pass)
  T *zout;               // storage-precision output (may be null)
  double *zout64;        // widened output (may be null)
  double *part;          // r.z tile partials (last pass, needs r64)
  unsigned long long *ovf_count;  // narrowing overflow (first pass, T=float)
  long long *ovf_first;
  T *resbuf;             // large-block path
  T *dbuf;
  SolverState *st;       // solve mode: gate + fused scalar step
  double *csum;          // solve mode: chunk sums of the two-level r.z sum (ChunkCtx)
  int want_branch;
  int prefetch;          // stream the first tiles' matrix data before the grid dependency wait
  int gate;              // 0: st->branch; 1: also skip when the fused update ran this first pass;
                         // 2: st->upd_branch (fused update: the step inside may change st->branch)
  int pdl;               // host side: launch with programmatic serialization
  WinSet win;            // z_in gather windows (passes after the first; n == 0: none)
  // offset-slot ("DIA") layout of stencil plans (k_bjac_dia; null: not available)
  const T *dval;             // values, slot k of row r at (r / 32) * 32 kDiaSlots + 32 k + r % 32
  const uint16_t *dmeta;     // per row: present slots | in-block slots << 8
  const T *dnear;            // slots kDiaDiag - 1 .. + 1 only, 3 per row in the same slice layout (null: some
                             // in-block entry sits elsewhere); read by the fused update's first pass
  int doff[8];               // column offset of slot k (doff[kDiaDiag] == 0), ascending
  int ibany;                 // slots that are in-block in at least one row
};

template <typename T>
__device__ __forceinline__ bool gated_off(const PassArgs<T> &a) {
  if (a.st == nullptr) return false;
  const int b = a.gate == 2 ? a.st->upd_branch : a.st->branch;
  return a.st->done || b != a.want_branch || (a.gate == 1 && a.st->z1_ok);
}

template <typename T>
__device__ __forceinline__ T narrow_checked(const PassArgs<T> &a, double r, int row, bool check_ovf) {
  const T v = narrow_or_copy<T>(r);
  if (sizeof(T) == 4 && check_ovf && a.ovf_count != nullptr && isinf(v) && isfinite(r)) {
    atomicAdd(a.ovf_count, 1ull);
    atomicMin(a.ovf_first, static_cast<long long>(row));
  }
  return v;
}

// block [blo, bhi) containing `row`; b holds nbk+1 absolute offsets
__device__ __forceinline__ void find_block_abs(const int *b, int nbk, int row, int &blo, int &bhi) {
  int L = 0, H = nbk;
  while (H - L > 1) {
    const int M = (L + H) >> 1;
    if (b[M] <= row) L = M; else H = M;
  }
  blo = b[L];
  bhi = b[L + 1];
}

// Generic row of a pass (no row pattern): scans its SELL entries with
// explicit block bounds.  Returns res; sets d.
template <typename T, bool FIRST>
__device__ __forceinline__ T generic_row_scan(const PassArgs<T> &a, int row, int base, int width, const int *col,
                                              const T *val, T rv, T &dd) {
  T az = T(0);
  dd = T(0);
  for (int j = 0; j < width; j++) {
    const int cj = col[base + 32 * j];
    if (cj < 0) continue;
    const T vj = val[base + 32 * j];
    if (!FIRST) az = add_rn(az, mul_rn(vj, __ldg(a.zin + cj)));
    if (cj == row) dd = vj;
  }
  return FIRST ? rv : sub_rn(rv, az);
}

template <typename T>
__device__ __forceinline__ T generic_row_sweep(const PassArgs<T> &a, const TileDesc &d, int row, int base, int width,
                                               const int *col, const T *val, const T *s_w) {
  int blo, bhi;
  find_block_abs(a.boff + d.bf, d.nbk, row, blo, bhi);
  T acc = T(0);
  for (int j = 0; j < width; j++) {
    const int cj = col[base + 32 * j];
    if (cj >= blo && cj < bhi) acc = add_rn(acc, mul_rn(val[base + 32 * j], s_w[cj - d.lo]));
  }
  return acc;
}

// One tile of a fused (non-first-only) pass, consumer threads only.  col /
// val / spp / mt are the shared stage or the global arrays offset to the
// tile (same indexing); r64t / rTt the tile's residual slice.
// ---- pass bodies: one consumer thread owns rows tid and tid + kConsumers ----
// (kRowsPerThread rows per thread halve the per-tile instruction overhead
// and give each thread two independent dependency chains; the tile sums keep
// the 256-lane order of include/mpbjac_order.h: value k of thread t is lane
// t + k * kConsumers.)

// Tile sum of kRowsPerThread values per consumer thread in the fixed order:
// virtual lane t + k kConsumers, virtual warps butterfly, warp 0 butterflies
// the kTileThreads/32 warp sums padded with +0.  Result valid in thread 0.
template <typename R, int RPT = kRowsPerThread>
__device__ __forceinline__ R tile_tree_rows(const R (&v)[RPT], R *ws, int bar) {
  constexpr int NC = kTileThreads / RPT;  // consumer threads
  constexpr int kWarps = NC / 32;
  R s[RPT];
#pragma unroll
  for (int k = 0; k < RPT; k++) s[k] = warp_bfly(v[k]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  named_sync(bar, NC);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < RPT; k++) ws[warp + k * kWarps] = s[k];
  }
  named_sync(bar, NC);
  R r = R(0);
  if (warp == 0) {
    r = lane < kTileThreads / 32 ? ws[lane] : R(0);
    r = warp_bfly(r);
  }
  return r;
}

// KS: slots of the longest row pattern (compile time, 7 for 7-point stencils);
// table entries past a pattern's length are 0, so gathers need no predicate.
template <typename T>
struct PassRow {
  T res, dd, w, zown;
  const int *P;  // pattern row
  int base, width, i0, i1;  // SELL slot of the row; in-block slots [i0, i1)
  uint16_t m;
  bool valid;
};

// A pass up to its first inner sweep for one row: res = r - A z_in (all
// slots, stored order), d, w = res / d (written to the tile's s_w).
// GEN: the plan has generic rows (no row pattern); false compiles their path out
// zb (windows): the stage base + tid * sizeof(T); z_in of slot u of pattern
// pid at zb + s_zoff[pid * KS + u], the row's own z_in at zb + s_zoff[kPatMax * KS]
template <typename T, bool FIRST, int KS, bool GEN, bool WIN = false>
__device__ __forceinline__ void pass_row_init(PassRow<T> &q, const PassArgs<T> &a, const TileDesc &d, int tid,
                                              const int *col, const T *val, const int *spp, const uint16_t *mt,
                                              const double *r64t, const T *rTt, const int *s_pat, T *s_w,
                                              const unsigned char *zb = nullptr, const int *s_zoff = nullptr) {
  const int row = d.lo + tid;
  q.res = T(0);
  q.dd = T(1);
  q.w = T(0);
  q.zown = T(0);
  q.P = s_pat;
  q.base = q.width = q.i0 = q.i1 = 0;
  q.m = kMetaGeneric;
  q.valid = row < d.hi;
  if (!q.valid) return;
  const int si = (row >> 5) - d.s0;
  const int sb = spp[si];
  q.width = (spp[si + 1] - sb) >> 5;
  q.base = sb - d.e0 + (row & 31);
  q.m = mt[tid];
  const T rv = r64t != nullptr ? narrow_checked(a, r64t[tid], row, FIRST) : rTt[tid];
  const T *zr = FIRST ? nullptr : a.zin + row;
  if (!FIRST) q.zown = (WIN && zb != nullptr) ? *reinterpret_cast<const T *>(zb + s_zoff[kPatMax * KS]) : __ldg(zr);
  if (!GEN || q.m != kMetaGeneric) {
    q.P = s_pat + meta_pid(q.m) * kPatStride;
    const int hdr = q.P[0], len = pat_len(hdr);
    q.i0 = meta_i0(q.m);
    q.i1 = meta_i1(q.m);
    T az = T(0);
    if (!FIRST) {
      T v[KS], g[KS];
      if (WIN && zb != nullptr) {
        const int *zo = s_zoff + meta_pid(q.m) * KS;
#pragma unroll
        for (int u = 0; u < KS; u++) {
          v[u] = u < len ? val[q.base + 32 * u] : T(0);
          g[u] = *reinterpret_cast<const T *>(zb + zo[u]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < KS; u++) {
          v[u] = u < len ? val[q.base + 32 * u] : T(0);
          g[u] = __ldg(zr + q.P[1 + u]);
        }
      }
#pragma unroll
      for (int u = 0; u < KS; u++)
        if (u < len) az = add_rn(az, mul_rn(v[u], g[u]));
    }
    q.dd = val[q.base + 32 * pat_dpos(hdr)];
    q.res = FIRST ? rv : sub_rn(rv, az);
  } else {
    q.res = generic_row_scan<T, FIRST>(a, row, q.base, q.width, col, val, rv, q.dd);
  }
  q.w = div_rn(q.res, q.dd);
  s_w[tid] = q.w;
}

// A_b w over the row's in-block entries (one inner sweep's sum)
template <typename T, bool GEN>
__device__ __forceinline__ T pass_row_sweep(const PassRow<T> &q, const PassArgs<T> &a, const TileDesc &d, int tid,
                                            const int *col, const T *val, const T *s_w) {
  T acc = T(0);
  if (!q.valid) return acc;
  if (!GEN || q.m != kMetaGeneric) {
#pragma unroll 1
    for (int j = q.i0; j < q.i1; j++) acc = add_rn(acc, mul_rn(val[q.base + 32 * j], s_w[tid + q.P[1 + j]]));
  } else {
    acc = generic_row_sweep(a, d, d.lo + tid, q.base, q.width, col, val, s_w);
  }
  return acc;
}

// One tile of a fused (non-first-only) pass, consumer threads only.  col /
// val / spp / mt are the shared stage or the global arrays offset to the
// tile (same indexing); r64t / rTt the tile's residual slice.
// Deferred tile sums (MPB_DEFER_TREE=1; off: C2 -0.3 %, but the C4 last pass
// +27 % and C3 / C5 +1 %): with inner sweeps, the
// warps store their warp sums of tile i and move on; warp 0 finishes tile
// i's sum after the first sweep barrier of the CTA's next tile (which every
// warp passes only after storing), so the tile sum needs no barriers of its
// own.  Same arithmetic as tile_tree_rows.  dt: the pending tile (-1 none)
// and the ws slot (0/1) it occupies.
#ifndef MPB_DEFER_TREE
#define MPB_DEFER_TREE 0
#endif
struct DeferredTree {
  int tile = -1, slot = 0;
};
__device__ __forceinline__ void deferred_tree_finish(DeferredTree &dt, double *part, const double *ws) {
  if (dt.tile < 0) return;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double r = lane < kTileThreads / 32 ? ws[dt.slot * 8 + lane] : 0.0;
    r = warp_bfly(r);
    if (lane == 0) put_part(part + dt.tile, r);
  }
  dt.tile = -1;
}

template <typename T, bool FIRST, bool LAST, int KS, bool GEN, int RPT = kRowsPerThread, bool WIN = false>
__device__ __forceinline__ void bjac_tile_body(const PassArgs<T> &a, int tile, const TileDesc &d, const int *col,
                                               const T *val, const int *spp, const uint16_t *mt, const double *r64t,
                                               const T *rTt, const int *s_pat, T *s_w, double *ws,
                                               DeferredTree &dt, const unsigned char *sb = nullptr,
                                               const int *s_zoff = nullptr) {
  const bool defer = MPB_DEFER_TREE && LAST && a.part != nullptr && a.t >= 2;
  constexpr int NC = kTileThreads / RPT;
  PassRow<T> q[RPT];
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    const int tid = threadIdx.x + k * NC;
    pass_row_init<T, FIRST, KS, GEN, WIN>(q[k], a, d, tid, col, val, spp, mt, r64t, rTt, s_pat, s_w,
                                          (WIN && sb != nullptr) ? sb + tid * sizeof(T) : nullptr, s_zoff);
  }
  for (int s = 1; s < a.t; s++) {  // inner sweeps, the tile's w in shared memory
    named_sync(kBarConsumers, NC);
    if (defer && s == 1) deferred_tree_finish(dt, a.part, ws);
    T acc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; k++)
      acc[k] = pass_row_sweep<T, GEN>(q[k], a, d, threadIdx.x + k * NC, col, val, s_w);
    named_sync(kBarConsumers, NC);
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      if (!q[k].valid) continue;
      q[k].w = add_rn(q[k].w, div_rn(sub_rn(q[k].res, acc[k]), q[k].dd));
      s_w[threadIdx.x + k * NC] = q[k].w;
    }
  }
  double prod[RPT];
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    prod[k] = 0.0;
    if (!q[k].valid) continue;
    const int tid = threadIdx.x + k * NC, row = d.lo + tid;
    const T zo = FIRST ? q[k].w : add_rn(q[k].zown, q[k].w);
    if (a.zout != nullptr) st_keep(a.zout + row, zo);
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) prod[k] = __dmul_rn(r64t[tid], static_cast<double>(zo));
  }
  if (defer) {
    dt.slot ^= 1;
#pragma unroll
    for (int k = 0; k < RPT; k++) {  // virtual warp (threadIdx.x >> 5) + k * NC / 32
      const double w = warp_bfly(prod[k]);
      if ((threadIdx.x & 31) == 0) ws[dt.slot * 8 + (threadIdx.x >> 5) + k * (NC / 32)] = w;
    }
    dt.tile = tile;
  } else if (LAST && a.part != nullptr) {
    const double tot = tile_tree_rows<double, RPT>(prod, ws, kBarConsumers);
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
  }
}

// First pass of a tile: z1 = D_b^{-1} r (bjac.py:134-136), reading only the
// in-block entries (plan's in-block SELL): y = r / d, then t-1 sweeps
// y += (r - A_b y) / d over the in-block entries in ascending column order.
// res[k]: row tid + k kConsumers's residual in T (valid rows).
template <typename T, bool GEN, int RPT = kRowsPerThread>
__device__ __forceinline__ void bjac_first_body(const PassArgs<T> &a, const TileDesc &d, const int *col,
                                                const T *val, const int *spp, const uint16_t *mt,
                                                const T (&res)[RPT], const int *s_pat, T *s_w) {
  constexpr int NC = kTileThreads / RPT;
  T dd[RPT], w[RPT];
  const int *P[RPT];
  int base[RPT], nib[RPT];
  bool pat[RPT], valid[RPT];
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    const int tid = threadIdx.x + k * NC, row = d.lo + tid;
    dd[k] = T(1);
    w[k] = T(0);
    P[k] = s_pat;
    base[k] = nib[k] = 0;
    pat[k] = true;
    valid[k] = row < d.hi;
    if (!valid[k]) continue;
    const int si = (row >> 5) - d.s0;
    const int sb = spp[si];
    base[k] = sb - d.ie0 + (row & 31);
    const uint16_t m = mt[tid];
    pat[k] = !GEN || m != kMetaGeneric;
    if (pat[k]) {
      const int i0 = meta_i0(m);
      nib[k] = meta_i1(m) - i0;
      dd[k] = val[base[k] + 32 * (pat_dpos(s_pat[meta_pid(m) * kPatStride]) - i0)];
      P[k] = s_pat + meta_pid(m) * kPatStride + 1 + i0;
    } else {
      const int iwidth = (spp[si + 1] - sb) >> 5;
      for (int j = 0; j < iwidth; j++) {
        const int cc = col[base[k] + 32 * j];
        if (cc < 0) break;
        nib[k] = j + 1;
        if (cc == row) dd[k] = val[base[k] + 32 * j];
      }
    }
    w[k] = div_rn(res[k], dd[k]);
    s_w[tid] = w[k];
  }
  for (int s = 1; s < a.t; s++) {
    named_sync(kBarConsumers, NC);
    T acc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      const int tid = threadIdx.x + k * NC;
      acc[k] = T(0);
      if (pat[k]) {
#pragma unroll 1
        for (int j = 0; j < nib[k]; j++) acc[k] = add_rn(acc[k], mul_rn(val[base[k] + 32 * j], s_w[tid + P[k][j]]));
      } else {
        for (int j = 0; j < nib[k]; j++)
          acc[k] = add_rn(acc[k], mul_rn(val[base[k] + 32 * j], s_w[col[base[k] + 32 * j] - d.lo]));
      }
    }
    named_sync(kBarConsumers, NC);
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      if (!valid[k]) continue;
      w[k] = add_rn(w[k], div_rn(sub_rn(res[k], acc[k]), dd[k]));
      s_w[threadIdx.x + k * NC] = w[k];
    }
  }
#pragma unroll
  for (int k = 0; k < RPT; k++) {
    if (!valid[k]) continue;
    const int row = d.lo + threadIdx.x + k * NC;
    if (a.zout != nullptr) st_keep(a.zout + row, w[k]);
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(w[k]);
  }
}

// Full staged tile of a pass after the first, pattern rows only, one row per
// consumer thread, tile start a multiple of 32 (so thread tid's row sits in
// the tile's slice tid / 32 at lane tid % 32): the same arithmetic as
// bjac_tile_body without its per-row validity branches, with the inner
// sweep unrolled to KI in-block entries.
// COH: z_in was written earlier in the same kernel (the wave kernel's update
// items): plain coherent loads instead of the read-only path.
template <typename T, bool LAST, int KS, int KI, bool WIN = false, bool COH = false>
__device__ __forceinline__ void bjac_tile_full(const PassArgs<T> &a, int tile, const TileDesc &d, const T *val,
                                               const int *spp, const uint16_t *mt, const double *r64t,
                                               const int *s_pat, T *s_w, double *ws,
                                               const unsigned char *sb = nullptr, const int *s_zoff = nullptr) {
  const int tid = threadIdx.x, row = d.lo + tid;
  const bool valid = row < d.hi;  // warp-uniform: tiles of a multiple of 32 rows
  const int ti = valid ? tid : 0;
  const int base = spp[ti >> 5] - d.e0 + (ti & 31);
  const uint16_t m = mt[ti];
  const int *P = s_pat + meta_pid(m) * kPatStride;
  const int hdr = P[0], len = pat_len(hdr);
  const T *zr = a.zin + d.lo + ti;
  T v[KS], g[KS], zown;
  if (WIN) {  // z_in from the stage's gather windows
    const unsigned char *zb = sb + tid * sizeof(T);
    const int *zo = s_zoff + meta_pid(m) * KS;
#pragma unroll
    for (int u = 0; u < KS; u++) {
      v[u] = val[base + 32 * u];
      g[u] = *reinterpret_cast<const T *>(zb + zo[u]);
    }
    zown = *reinterpret_cast<const T *>(zb + s_zoff[kPatMax * KS]);
  } else {
#pragma unroll
    for (int u = 0; u < KS; u++) {
      v[u] = val[base + 32 * u];       // slots past len: never summed (the stage extends past them)
      g[u] = COH ? zr[P[1 + u]] : __ldg(zr + P[1 + u]);  // table offsets past len are 0
    }
    zown = COH ? *zr : __ldg(zr);
  }
  T az = T(0);
#pragma unroll
  for (int u = 0; u < KS; u++)
    if (u < len) az = add_rn(az, mul_rn(v[u], g[u]));
  const T dd = val[base + 32 * pat_dpos(hdr)];
  const T res = sub_rn(narrow_or_copy<T>(r64t[ti]), az);
  T w = div_rn(res, dd);
  s_w[tid] = w;  // (rows past the tile: never read by the tile's rows)
  const int i0 = meta_i0(m), i1 = meta_i1(m);
  for (int s = 1; s < a.t; s++) {
    named_sync(kBarConsumers, kTileThreads);
    T acc = T(0);
#pragma unroll
    for (int j = 0; j < KI; j++) {
      const int jj = i0 + j;
      if (jj < i1) acc = add_rn(acc, mul_rn(val[base + 32 * jj], s_w[tid + P[1 + jj]]));
    }
    named_sync(kBarConsumers, kTileThreads);
    w = add_rn(w, div_rn(sub_rn(res, acc), dd));
    s_w[tid] = w;
  }
  const T zo = add_rn(zown, w);
  if (valid && a.zout != nullptr) st_keep(a.zout + row, zo);
  if (valid && a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
  if (LAST && a.part != nullptr) {
    double prod[1] = {valid ? __dmul_rn(r64t[ti], static_cast<double>(zo)) : 0.0};
    const double tot = tile_tree_rows<double, 1>(prod, ws, kBarConsumers);
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
  }
}

// Warp-per-block tile of a pass after the first (kernels with 4 consumer
// warps, RPT = 2): the partition's blocks all have 64 rows, so block w of the
// tile is rows [lo + 64 w, lo + 64 w + 64) and consumer warp w owns it, two
// rows per lane (tile rows 64 w + lane and 64 w + 32 + lane: SELL slices 2 w
// and 2 w + 1).  In-block neighbours never leave the warp's rows, so the inner
// sweeps synchronise with __syncwarp only and the consumer warps of a CTA run
// their blocks independently -- no CTA-wide barrier per sweep or per tile sum.
// The tile's r.z sum keeps the order of include/mpbjac_order.h: virtual warp
// 2 w + k butterflies rows 64 w + 32 k .. + 31 into wsum[2 w + k]; the warp
// that arrives last on the stage's counter butterflies the 8 warp sums padded
// with +0.  Same arithmetic per row as bjac_tile_full.
template <typename T, bool LAST, int KS, int KI>
__device__ __forceinline__ void bjac_tile_wb(const PassArgs<T> &a, int tile, const TileDesc &d, const T *val,
                                             const int *spp, const uint16_t *mt, const double *r64t,
                                             const int *s_pat, T *s_w, double *wsum, unsigned int *wcnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool active = 64 * warp < d.hi - d.lo;  // warp-uniform: the tile holds (hi - lo) / 64 blocks
  double s[2] = {0.0, 0.0};
  if (active) {
    int ti[2], base[2], i0[2], i1[2];
    const int *P[2];
    T v[2][KS], g[2][KS], zown[2], res[2], dd[2], w[2];
    int len[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      ti[k] = 64 * warp + 32 * k + lane;
      base[k] = spp[2 * warp + k] - d.e0 + lane;
      const uint16_t m = mt[ti[k]];
      P[k] = s_pat + meta_pid(m) * kPatStride;
      i0[k] = meta_i0(m);
      i1[k] = meta_i1(m);
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const T *zr = a.zin + d.lo + ti[k];
#pragma unroll
      for (int u = 0; u < KS; u++) {
        v[k][u] = val[base[k] + 32 * u];       // slots past len: never summed
        g[k][u] = __ldg(zr + P[k][1 + u]);     // table offsets past len are 0
      }
      zown[k] = __ldg(zr);
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int hdr = P[k][0];
      len[k] = pat_len(hdr);
      T az = T(0);
#pragma unroll
      for (int u = 0; u < KS; u++)
        if (u < len[k]) az = add_rn(az, mul_rn(v[k][u], g[k][u]));
      dd[k] = val[base[k] + 32 * pat_dpos(hdr)];
      res[k] = sub_rn(narrow_or_copy<T>(r64t[ti[k]]), az);
      w[k] = div_rn(res[k], dd[k]);
      s_w[ti[k]] = w[k];
    }
    for (int sw = 1; sw < a.t; sw++) {
      __syncwarp();
      T acc[2];
#pragma unroll
      for (int k = 0; k < 2; k++) {
        acc[k] = T(0);
#pragma unroll
        for (int j = 0; j < KI; j++) {
          const int jj = i0[k] + j;
          if (jj < i1[k]) acc[k] = add_rn(acc[k], mul_rn(val[base[k] + 32 * jj], s_w[ti[k] + P[k][1 + jj]]));
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2; k++) {
        w[k] = add_rn(w[k], div_rn(sub_rn(res[k], acc[k]), dd[k]));
        s_w[ti[k]] = w[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int row = d.lo + ti[k];
      const T zo = add_rn(zown[k], w[k]);
      if (a.zout != nullptr) st_keep(a.zout + row, zo);
      if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
      if (LAST && a.part != nullptr) s[k] = __dmul_rn(r64t[ti[k]], static_cast<double>(zo));
    }
  }
  if (LAST && a.part != nullptr) {
    const double tot2 = warp_bfly2(s[0], s[1]);
    if ((lane & 15) == 0) wsum[2 * warp + (lane >> 4)] = tot2;
    __syncwarp();
    unsigned int old = 0;
    if (lane == 0)
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(wcnt)) : "memory");
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == kTileThreads / 64 - 1) {  // the tile's last warp: every warp sum is stored
      double r = lane < kTileThreads / 32 ? wsum[lane] : 0.0;
      r = warp_bfly(r);
      if (lane == 0) {
        *wcnt = 0u;
        put_part(a.part + tile, r);
      }
    }
  }
}

template <typename T, bool FIRST, bool R64>
__host__ __device__ inline StageLayout bjac_layout(const TileGeom &g) {
  // v0: the residual slice
  return stage_layout(g.cap_e, sizeof(T), g.max_sl, g.cols != 0, true, R64 ? 8 : sizeof(T), 0, 0);
}
// the same plus the z_in gather windows (passes after the first)
template <typename T, bool FIRST, bool R64>
__host__ __device__ inline StageLayout bjac_layout_win(const TileGeom &g, const WinSet &w) {
  StageLayout L = bjac_layout<T, FIRST, R64>(g);
  L.win = L.bytes;
  L.bytes += win_off(w, w.n, sizeof(T));
  return L;
}

// Per-CTA table of gather byte offsets (relative to stage base + tid * es):
// s_zoff[pid * KS + u] for slot u of pattern pid (slots past the pattern's
// length point at the row's own z_in), s_zoff[kPatMax * KS] for the row itself.
template <typename T, int KS>
__device__ __forceinline__ void load_zoff(int *s_zoff, const int *pat, int npat, const WinSet &w,
                                          const StageLayout &L) {
  constexpr int es = sizeof(T);
  auto zoff = [&](int o) {
    int k = 0;
    while (k + 1 < w.n && o > w.b[k]) k++;
    return static_cast<int>(L.win + win_off(w, k, es)) - floor16i(w.a[k] * es) + o * es;
  };
  for (int idx = threadIdx.x; idx <= npat * KS; idx += blockDim.x) {
    if (idx == npat * KS) {
      s_zoff[kPatMax * KS] = zoff(0);
      continue;
    }
    const int q = idx / KS, u = idx % KS;
    const int hdr = __ldg(pat + q * kPatStride);
    s_zoff[idx] = zoff(u < pat_len(hdr) ? __ldg(pat + q * kPatStride + 1 + u) : 0);
  }
}

// Persistent, warp-specialised fused pass.  TWO: the two-level dot-sum order
// (chunk owners in the producer warp); false compiles that machinery out.
// RPT: tile rows per consumer thread (kTileThreads / RPT consumer threads +
// the producer warp per CTA)
// WIN: z_in gathered from the stage's gather windows (passes after the first,
// plans with windows; a.win.n > 0)
// MPB_MINB_LAST=n (experiment): compile the BJAC tile kernels for n co-resident CTAs per SM
#ifdef MPB_MINB_LAST
#define MPB_TILE_BOUNDS(RPT) __launch_bounds__(kTileThreads / RPT + 32, MPB_MINB_LAST)
#else
#define MPB_TILE_BOUNDS(RPT) __launch_bounds__(kTileThreads / RPT + 32)
#endif
template <typename T, bool FIRST, bool LAST, bool R64, int KS, bool GEN, bool TWO = false, int RPT = kRowsPerThread,
          bool WIN = false>
__global__ void MPB_TILE_BOUNDS(RPT) k_bjac_tile(const PassArgs<T> a) {
  constexpr int NC = kTileThreads / RPT;
  constexpr int kFinRpt = NC >= kFinThreads ? 1 : kFinThreads / NC;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ T s_w[kTileRows];
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  __shared__ int s_zoff[WIN ? kPatMax * KS + 1 : 1];
  // warp-per-block tiles (bjac_tile_wb): per-stage warp sums and arrival counters
  constexpr bool kWb = !FIRST && !GEN && RPT == 2 && R64 && !WIN && !MPB_DEFER_TREE;
  __shared__ double s_wsum[kWb ? kMaxStages * (kTileThreads / 32) : 1];
  __shared__ unsigned int s_wcnt[kMaxStages];
  if (threadIdx.x < kMaxStages) s_wcnt[threadIdx.x] = 0u;  // (published by ring_init's barrier)
#ifdef MPB_TIMELINE
  const unsigned long long t_entry = globaltimer_now();
#endif
  const int ns = a.g.ns;
  constexpr bool kIB = FIRST && !LAST;  // first pass alone: in-block entries only
  static_assert(!(WIN && FIRST), "gather windows serve the passes after the first");
  const StageLayout L = WIN ? bjac_layout_win<T, FIRST, R64>(a.g, a.win) : bjac_layout<T, FIRST, R64>(a.g);
  load_patterns(s_pat, a.pat, a.g.npat);
  if (WIN) load_zoff<T, KS>(s_zoff, a.pat, a.g.npat, a.win, L);
  ring_init(R, ns, NC);
  if (threadIdx.x >= NC) {  // producer warp
    using RT = typename std::conditional<R64, double, T>::type;
    const RT *rsrc = R64 ? reinterpret_cast<const RT *>(a.r64) : reinterpret_cast<const RT *>(a.rT);
    const ChunkCtx ck{(TWO && LAST && a.part != nullptr && a.st != nullptr) ? a.csum : nullptr, a.part, a.g.ntiles,
                      TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      if (kIB)
        produce<T, RT, uint8_t, uint8_t, true>(R, st, a.td, tile, a.g, L, smem + st * L.bytes, a.ib_sp, a.ib_col,
                                               a.ib_val, a.meta, rsrc, nullptr, nullptr,
                                               static_cast<const uint8_t *>(nullptr), part);
      else
        produce<T, RT, uint8_t, uint8_t>(R, st, a.td, tile, a.g, L, smem + st * L.bytes, a.sp, a.scol, a.sval,
                                         a.meta, rsrc, nullptr, nullptr, static_cast<const uint8_t *>(nullptr), part,
                                         WIN ? &a.win : nullptr, a.zin);
    };
    auto gated = [&]() { return gated_off(a); };
    if (TWO && ck.csum != nullptr && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == NC)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td);
    else
      pdl_wait();
    if (gated_off(a)) return;
  } else {
    pdl_wait();
    if (gated_off(a)) return;
    if (LAST && threadIdx.x == 0) {
      tl_mark(a.st, 0, 0, false);
#ifdef MPB_TIMELINE
      tl_mark_at(a.st, 3, 0, false, t_entry);
      tl_mark_at(a.st, 3, 1, true, t_entry);
      tl_mark(a.st, 3, 3, true);
#endif
    }
    DeferredTree dt;
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * L.bytes;
      const bool ok = R.ok[st] != 0;
      const bool scols = ok && a.g.cols && d.ngen > 0;
      if (kIB) {
        const int *col = scols ? reinterpret_cast<const int *>(sb + L.col) : a.ib_col + d.ie0;
        T rv[RPT];
#pragma unroll
        for (int k = 0; k < RPT; k++) {
          const int tid = threadIdx.x + k * NC, row = d.lo + tid;
          rv[k] = T(0);
          if (row >= d.hi) continue;
          if (R64) rv[k] = narrow_checked(a, ok ? staged(sb + L.v0, a.r64, d.lo, d.hi)[tid] : a.r64[row], row, true);
          else rv[k] = ok ? staged(sb + L.v0, a.rT, d.lo, d.hi)[tid] : a.rT[row];
        }
        if (ok) {
          bjac_first_body<T, GEN, RPT>(a, d, col, reinterpret_cast<const T *>(sb + L.val),
                             staged(sb + L.sp, a.ib_sp, d.s0, d.s1 + 1), staged(sb + L.meta, a.meta, d.lo, d.hi), rv,
                             s_pat, s_w);
        } else {
          bjac_first_body<T, GEN, RPT>(a, d, col, a.ib_val + d.ie0, a.ib_sp + d.s0, a.meta + d.lo, rv, s_pat, s_w);
        }
      } else {
        const int *col = scols ? reinterpret_cast<const int *>(sb + L.col) : a.scol + d.e0;
        constexpr bool kFast = !FIRST && !GEN && RPT == 1 && R64 && !MPB_DEFER_TREE;
        if (kWb && ok && a.g.ub == 64 && ((d.hi - d.lo) & 63) == 0 && (d.lo & 63) == 0 && a.g.kib <= 7) {
          const T *val = reinterpret_cast<const T *>(sb + L.val);
          const int *spp = staged(sb + L.sp, a.sp, d.s0, d.s1 + 1);
          const uint16_t *mt = staged(sb + L.meta, a.meta, d.lo, d.hi);
          const double *r64t = staged(sb + L.v0, a.r64, d.lo, d.hi);
          if (a.g.kib <= 3)
            bjac_tile_wb<T, LAST, KS, 3>(a, tile, d, val, spp, mt, r64t, s_pat, s_w, s_wsum + st * (kTileThreads / 32),
                                         s_wcnt + st);
          else
            bjac_tile_wb<T, LAST, KS, 7>(a, tile, d, val, spp, mt, r64t, s_pat, s_w, s_wsum + st * (kTileThreads / 32),
                                         s_wcnt + st);
        } else if (kFast && ok && kFastTiles && ((d.hi - d.lo) & 31) == 0 && (d.lo & 31) == 0 && a.g.kib <= 7) {
          const T *val = reinterpret_cast<const T *>(sb + L.val);
          const int *spp = staged(sb + L.sp, a.sp, d.s0, d.s1 + 1);
          const uint16_t *mt = staged(sb + L.meta, a.meta, d.lo, d.hi);
          const double *r64t = staged(sb + L.v0, a.r64, d.lo, d.hi);
          if (a.g.kib <= 3)
            bjac_tile_full<T, LAST, KS, 3, WIN>(a, tile, d, val, spp, mt, r64t, s_pat, s_w, ws, sb, s_zoff);
          else
            bjac_tile_full<T, LAST, KS, 7, WIN>(a, tile, d, val, spp, mt, r64t, s_pat, s_w, ws, sb, s_zoff);
        } else if (ok) {
          bjac_tile_body<T, FIRST, LAST, KS, GEN, RPT, WIN>(a, tile, d, col, reinterpret_cast<const T *>(sb + L.val),
                                             staged(sb + L.sp, a.sp, d.s0, d.s1 + 1),
                                             staged(sb + L.meta, a.meta, d.lo, d.hi),
                                             R64 ? staged(sb + L.v0, a.r64, d.lo, d.hi) : nullptr,
                                             R64 ? nullptr : staged(sb + L.v0, a.rT, d.lo, d.hi), s_pat, s_w, ws, dt,
                                             sb, s_zoff);
        } else {
          bjac_tile_body<T, FIRST, LAST, KS, GEN, RPT>(a, tile, d, col, a.sval + d.e0, a.sp + d.s0, a.meta + d.lo,
                                             R64 ? a.r64 + d.lo : nullptr, R64 ? nullptr : a.rT + d.lo, s_pat, s_w,
                                             ws, dt);
        }
      }
      ring_release(R, st);
    }
    if (dt.tile >= 0) {  // the last tile's deferred sum: every warp has stored its share
      named_sync(kBarConsumers, NC);
      deferred_tree_finish(dt, a.part, ws);
    }
    if (LAST && threadIdx.x == 0) tl_mark(a.st, 0, 1, true);
  }
  pdl_trigger();  // dependents may launch into the SMs this grid drains
  if (LAST && a.part != nullptr)
    finish_grid<16, kFinRpt>(a.st, 0, kStepRho, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---------------------------------------------------------------------------
// Offset-slot pass after the first, warp per 64-row block (k_bjac_dia).
//
// For plans whose row patterns all draw their column offsets from the same
// kDiaSlots offsets (7-point stencils) and whose blocks all have 64 rows.
// The pass streams the offset-slot value array (PassArgs::dval) instead of
// the SELL values: no slice pointers, no pattern ids, no pattern-table
// lookups and no dynamic slot indices -- a row's slot k is at a fixed
// shared-memory offset, its column is row + doff[k] (kernel constants), its
// diagonal is slot kDiaDiag, and what the row has / which of it is in-block
// is one 16-bit mask.  Consumer warp w owns block w of the tile, two rows
// per lane (bjac_tile_wb's mapping and tile-sum order); the arithmetic per
// row is bjac_tile_full's: res = r - sum over present slots in ascending
// slot (= stored) order, w = res / d, t - 1 masked sweeps, z = z_in + w.
// IBM: slots that may be in-block (compile time; others are never tested).
// ---------------------------------------------------------------------------
// v is "defined" without an instruction: its value is whatever the register
// held.  For operands that are only used under the same predicate as their
// real definition (saves the zero-initialising move per predicated load).
__device__ __forceinline__ void undefined_value(float &v) { asm volatile("" : "=f"(v)); }
__device__ __forceinline__ void undefined_value(double &v) { asm volatile("" : "=d"(v)); }

template <typename T>
__host__ __device__ constexpr uint32_t dia_stage_bytes() {
  return kTileRows * kDiaSlots * sizeof(T) + kTileRows * 2u + kTileRows * 8u;  // values, masks, fp64 residual
}

template <typename T, bool LAST, int IBM>
__device__ __forceinline__ void dia_tile_wb(const PassArgs<T> &a, const int (&off)[kDiaSlots], int tile, int lo,
                                            int nrows, const T *val, const uint16_t *dm, const double *r64t,
                                            T *s_w, double *wsum, unsigned int *wcnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool active = 64 * warp < nrows;  // warp-uniform: the tile holds nrows / 64 blocks
  double s[2] = {0.0, 0.0};
  if (active) {
    T v[2][kDiaSlots], g[2][kDiaSlots], res[2], w[2];
    unsigned int m[2];
    int ti[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      ti[k] = 64 * warp + 32 * k + lane;
      m[k] = dm[ti[k]];
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const T *vb = val + (2 * warp + k) * (32 * kDiaSlots) + lane;
      const T *zr = a.zin + lo + ti[k];
#pragma unroll
      for (int u = 0; u < kDiaSlots; u++) {
        v[k][u] = vb[32 * u];
        undefined_value(g[k][u]);  // (an absent slot's product is computed and never added)
        if ((m[k] >> u) & 1u) g[k][u] = __ldg(zr + off[u]);
      }
    }
    // (a warp-uniform branch to an unpredicated body for 32-row groups whose rows have all
    // slots measured slower: 30.5 us against 28.9 us on C2)
#pragma unroll
    for (int k = 0; k < 2; k++) {
      T az = T(0);
#pragma unroll
      for (int u = 0; u < kDiaSlots; u++)
        if ((m[k] >> u) & 1u) az = add_rn(az, mul_rn(v[k][u], g[k][u]));
      res[k] = sub_rn(narrow_or_copy<T>(r64t[ti[k]]), az);
      w[k] = div_rn(res[k], v[k][kDiaDiag]);
      s_w[ti[k]] = w[k];
    }
    for (int sw = 1; sw < a.t; sw++) {
      __syncwarp();
      T acc[2];
#pragma unroll
      for (int k = 0; k < 2; k++) {
        acc[k] = T(0);
#pragma unroll
        for (int u = 0; u < kDiaSlots; u++)
          if ((IBM >> u) & 1) {
            // acc is never -0 (it starts at +0), so adding +0 for a slot that is not in-block changes nothing
            const bool in = (m[k] >> (8 + u)) & 1u;
            T sv;
            undefined_value(sv);
            if (in) sv = s_w[ti[k] + off[u]];
            acc[k] = add_rn(acc[k], in ? mul_rn(v[k][u], sv) : T(0));
          }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2; k++) {
        w[k] = add_rn(w[k], div_rn(sub_rn(res[k], acc[k]), v[k][kDiaDiag]));
        s_w[ti[k]] = w[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int row = lo + ti[k];
      const T zo = add_rn(g[k][kDiaDiag], w[k]);  // (the diagonal's gather is the row's own z_in)
      if (a.zout != nullptr) st_keep(a.zout + row, zo);
      if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
      if (LAST && a.part != nullptr) s[k] = __dmul_rn(r64t[ti[k]], static_cast<double>(zo));
    }
  }
  if (LAST && a.part != nullptr) {
    const double tot2 = warp_bfly2(s[0], s[1]);
    if ((lane & 15) == 0) wsum[2 * warp + (lane >> 4)] = tot2;
    __syncwarp();
    unsigned int old = 0;
    if (lane == 0)
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(wcnt)) : "memory");
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == kTileThreads / 64 - 1) {  // the tile's last warp: every warp sum is stored
      double r = lane < kTileThreads / 32 ? wsum[lane] : 0.0;
      r = warp_bfly(r);
      if (lane == 0) {
        *wcnt = 0u;
        put_part(a.part + tile, r);
      }
    }
  }
}

// (no minimum CTA count: 7 CTAs per SM at 56 registers measured 30.9 us against 28.9 us at
// ptxas' own 64 registers / 6 CTAs on C2; the fused update showed no difference at 6)
template <typename T, bool LAST, bool TWO, int IBM>
__global__ void __launch_bounds__(kTileThreads / 2 + 32) k_bjac_dia(const PassArgs<T> a) {
  constexpr int NC = kTileThreads / 2;
  constexpr int kFinRpt = NC >= kFinThreads ? 1 : kFinThreads / NC;
  constexpr uint32_t kVal = kTileRows * kDiaSlots * sizeof(T), kMeta = kTileRows * 2u;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ T s_w[kTileRows];
  __shared__ double ws[32];
  __shared__ double s_wsum[kMaxStages * (kTileThreads / 32)];
  __shared__ unsigned int s_wcnt[kMaxStages];
  if (threadIdx.x < kMaxStages) s_wcnt[threadIdx.x] = 0u;  // (published by ring_init's barrier)
  const int ns = a.g.ns;
  ring_init(R, ns, NC);
  const bool red = LAST && a.g.red != 0 && a.part != nullptr && a.st != nullptr;
  if (red && blockIdx.x == 0) {  // this CTA takes no tiles: its first warp streams the r.z sum
    pdl_wait();
    if (!gated_off(a) && threadIdx.x < 32) reduce_stream(a.st, kStepRho, a.part, a.g.ntiles);
    pdl_trigger();
    return;
  }
  if (threadIdx.x >= NC) {  // producer warp
    const ChunkCtx ck{(TWO && LAST && a.part != nullptr && a.st != nullptr) ? a.csum : nullptr, a.part, a.g.ntiles,
                      TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      TileDesc d;
      if (part != kFillDynamic) {
        d = a.td[tile];
        R.desc[st] = d;
        R.ok[st] = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      } else {
        d = R.desc[st];
      }
      const uint32_t rows = static_cast<uint32_t>(d.hi - d.lo);  // a multiple of 64
      const uint32_t sbytes = rows * (kDiaSlots * static_cast<uint32_t>(sizeof(T)) + 2u), dbytes = rows * 8u;
      unsigned char *stage = smem + st * dia_stage_bytes<T>();
      if (part == kFillAll) mbar_arrive_expect_tx(&R.full[st], sbytes + dbytes);
      if (part == kFillStatic) mbar_expect_tx(&R.full[st], sbytes);
      if (part != kFillDynamic) {
        bulk_g2s_stream(stage, a.dval + static_cast<long long>(kDiaSlots) * d.lo,
                        rows * kDiaSlots * static_cast<uint32_t>(sizeof(T)), &R.full[st]);
        bulk_g2s(stage + kVal, a.dmeta + d.lo, rows * 2u, &R.full[st]);
      }
      if (part == kFillStatic) return;
      if (part == kFillDynamic) mbar_arrive_expect_tx(&R.full[st], dbytes);
      bulk_g2s(stage + kVal + kMeta, a.r64 + d.lo, dbytes, &R.full[st]);
    };
    auto gated = [&]() { return gated_off(a); };
    if (TWO && ck.csum != nullptr && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == NC)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td, gridDim.x - (red ? 1u : 0u));
    else
      pdl_wait();
    if (gated_off(a)) return;
  } else {
    pdl_wait();
    if (gated_off(a)) return;
    if (LAST && threadIdx.x == 0) tl_mark(a.st, 0, 0, false);
    int off[kDiaSlots];  // the slot offsets, register-resident (not re-read from the parameter bank per gather)
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++) {
      off[u] = a.doff[u];
      asm volatile("" : "+r"(off[u]));
    }
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const int lo = R.desc[st].lo, nrows = R.desc[st].hi - lo;
      const unsigned char *sb = smem + st * dia_stage_bytes<T>();
      dia_tile_wb<T, LAST, IBM>(a, off, tile, lo, nrows, reinterpret_cast<const T *>(sb),
                                reinterpret_cast<const uint16_t *>(sb + kVal),
                                reinterpret_cast<const double *>(sb + kVal + kMeta), s_w,
                                s_wsum + st * (kTileThreads / 32), s_wcnt + st);
      ring_release(R, st);
    }
    if (LAST && threadIdx.x == 0) tl_mark(a.st, 0, 1, true);
  }
  pdl_trigger();  // dependents may launch into the SMs this grid drains
  if (LAST && a.part != nullptr && !red)
    finish_grid<16, kFinRpt>(a.st, 0, kStepRho, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---------------------------------------------------------------------------
// Fused x/r update + next first pass in the offset-slot layout, warp per
// 64-row block (k_update_first's arithmetic; dia_tile_wb's mapping).  The
// first pass reads only in-block entries, here slots kDiaDiag - 1 .. + 1
// (PassArgs::dnear, 3 values per row): plans whose in-block entries are the
// diagonal and its two neighbours in the offset list.  No CTA barrier: the
// r.r tile sum uses the stage's arrival counter, the sweeps __syncwarp.
// ---------------------------------------------------------------------------
constexpr int kNearSlots = 3;
template <typename T>
__host__ __device__ constexpr uint32_t dia_uf_stage_bytes() {
  return kTileRows * kNearSlots * sizeof(T) + kTileRows * 2u + 4u * kTileRows * 8u;  // values, masks, r x p q
}

template <typename T>
__device__ __forceinline__ void dia_update_first_wb(const PassArgs<T> &a, int offm, int offp, int tile, int lo,
                                                    int nrows, double alpha, double *x, double *r, const T *val,
                                                    const uint16_t *dm, const double *rs, const double *xs,
                                                    const double *ps, const double *qs, T *s_w, double *wsum,
                                                    unsigned int *wcnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool active = 64 * warp < nrows;
  double sq[2] = {0.0, 0.0};
  if (active) {
    T v[2][kNearSlots], rv[2], w[2];
    unsigned int m[2];
    int ti[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      ti[k] = 64 * warp + 32 * k + lane;
      const int row = lo + ti[k];
      m[k] = dm[ti[k]] >> (8 + kDiaDiag - 1);  // in-block bits of the three near slots
      const T *vb = val + (2 * warp + k) * (32 * kNearSlots) + lane;
#pragma unroll
      for (int u = 0; u < kNearSlots; u++) v[k][u] = vb[32 * u];
      st_evict_first(x + row, __dadd_rn(xs[ti[k]], __dmul_rn(alpha, ps[ti[k]])));  // (read again by the next update only)
      const double rn = __dsub_rn(rs[ti[k]], __dmul_rn(alpha, qs[ti[k]]));
      r[row] = rn;
      sq[k] = __dmul_rn(rn, rn);
      rv[k] = narrow_checked(a, rn, row, true);
      w[k] = div_rn(rv[k], v[k][1]);
      s_w[ti[k]] = w[k];
    }
    for (int sw = 1; sw < a.t; sw++) {
      __syncwarp();
      T acc[2];
#pragma unroll
      for (int k = 0; k < 2; k++) {
        // acc is never -0 (it starts at +0), so adding +0 for a slot that is not in-block changes nothing
        T sm, sp;
        undefined_value(sm);
        undefined_value(sp);
        if (m[k] & 1u) sm = s_w[ti[k] + offm];
        if (m[k] & 4u) sp = s_w[ti[k] + offp];
        acc[k] = add_rn(T(0), (m[k] & 1u) ? mul_rn(v[k][0], sm) : T(0));
        acc[k] = add_rn(acc[k], (m[k] & 2u) ? mul_rn(v[k][1], w[k]) : T(0));  // (the row's own w)
        acc[k] = add_rn(acc[k], (m[k] & 4u) ? mul_rn(v[k][2], sp) : T(0));
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2; k++) {
        w[k] = add_rn(w[k], div_rn(sub_rn(rv[k], acc[k]), v[k][1]));
        s_w[ti[k]] = w[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int row = lo + ti[k];
      if (a.zout != nullptr) st_keep(a.zout + row, w[k]);
      if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(w[k]);
    }
  }
  {
    const double tot2 = warp_bfly2(sq[0], sq[1]);
    if ((lane & 15) == 0) wsum[2 * warp + (lane >> 4)] = tot2;
  }
  __syncwarp();
  unsigned int old = 0;
  if (lane == 0)
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(wcnt)) : "memory");
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old == kTileThreads / 64 - 1) {  // the tile's last warp: every warp sum is stored
    double t = lane < kTileThreads / 32 ? wsum[lane] : 0.0;
    t = warp_bfly(t);
    if (lane == 0) {
      *wcnt = 0u;
      put_part(a.part + tile, t);
    }
  }
}

template <typename T, bool TWO>
__global__ void __launch_bounds__(kTileThreads / 2 + 32)
    k_update_first_dia(const PassArgs<T> a, double *x, const double *p, const double *q, double *r) {
  constexpr int NC = kTileThreads / 2;
  constexpr int kFinRpt = NC >= kFinThreads ? 1 : kFinThreads / NC;
  constexpr uint32_t kVal = kTileRows * kNearSlots * sizeof(T), kMeta = kTileRows * 2u, kVec = kTileRows * 8u;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ T s_w[kTileRows];
  __shared__ double ws[32];
  __shared__ double s_wsum[kMaxStages * (kTileThreads / 32)];
  __shared__ unsigned int s_wcnt[kMaxStages];
  if (threadIdx.x < kMaxStages) s_wcnt[threadIdx.x] = 0u;  // (published by ring_init's barrier)
  const int ns = a.g.ns;
  ring_init(R, ns, NC);
  const bool red = a.g.red != 0;
  if (red && blockIdx.x == 0) {  // this CTA takes no tiles: its first warp streams the r.r sum
    pdl_wait();
    if (!gated_off(a) && threadIdx.x < 32) reduce_stream(a.st, kStepRrZ, a.part, a.g.ntiles);
    pdl_trigger();
    return;
  }
  if (threadIdx.x >= NC) {  // producer warp
    const ChunkCtx ck{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      TileDesc d;
      if (part != kFillDynamic) {
        d = a.td[tile];
        R.desc[st] = d;
        R.ok[st] = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      } else {
        d = R.desc[st];
      }
      const uint32_t rows = static_cast<uint32_t>(d.hi - d.lo);  // a multiple of 64
      const uint32_t vb = rows * kNearSlots * static_cast<uint32_t>(sizeof(T));
      const uint32_t sbytes = vb + rows * 2u, dbytes = 4u * rows * 8u;
      unsigned char *stage = smem + st * dia_uf_stage_bytes<T>();
      if (part == kFillAll) mbar_arrive_expect_tx(&R.full[st], sbytes + dbytes);
      if (part == kFillStatic) mbar_expect_tx(&R.full[st], sbytes);
      if (part != kFillDynamic) {
        bulk_g2s_stream(stage, a.dnear + static_cast<long long>(kNearSlots) * d.lo, vb, &R.full[st]);
        bulk_g2s(stage + kVal, a.dmeta + d.lo, rows * 2u, &R.full[st]);
      }
      if (part == kFillStatic) return;
      if (part == kFillDynamic) mbar_arrive_expect_tx(&R.full[st], dbytes);
      unsigned char *vec = stage + kVal + kMeta;
      bulk_g2s(vec, r + d.lo, rows * 8u, &R.full[st]);
      bulk_g2s_stream(vec + kVec, x + d.lo, rows * 8u, &R.full[st]);  // x and q: not read again before the next update
      bulk_g2s(vec + 2 * kVec, p + d.lo, rows * 8u, &R.full[st]);
      bulk_g2s_stream(vec + 3 * kVec, q + d.lo, rows * 8u, &R.full[st]);
    };
    auto gated = [&]() { return gated_off(a); };
    if (TWO && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == NC)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td, gridDim.x - (red ? 1u : 0u));
    else
      pdl_wait();
    if (gated_off(a)) return;
  } else {
    pdl_wait();
    if (gated_off(a)) return;
    if (threadIdx.x == 0) tl_mark(a.st, 2, 0, false);
    const double alpha = a.st->alpha;
    const int offm = a.doff[kDiaDiag - 1], offp = a.doff[kDiaDiag + 1];
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const int lo = R.desc[st].lo, nrows = R.desc[st].hi - lo;
      const unsigned char *sb = smem + st * dia_uf_stage_bytes<T>();
      const double *vec = reinterpret_cast<const double *>(sb + kVal + kMeta);
      dia_update_first_wb<T>(a, offm, offp, tile, lo, nrows, alpha, x, r, reinterpret_cast<const T *>(sb),
                             reinterpret_cast<const uint16_t *>(sb + kVal), vec, vec + kTileRows,
                             vec + 2 * kTileRows, vec + 3 * kTileRows, s_w, s_wsum + st * (kTileThreads / 32),
                             s_wcnt + st);
      ring_release(R, st);
    }
    if (threadIdx.x == 0) tl_mark(a.st, 2, 1, true);
  }
  pdl_trigger();
  if (!red) finish_grid<16, kFinRpt>(a.st, 2, kStepRrZ, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---------------------------------------------------------------------------
// Large blocks (a block spans several tiles, e.g. the reference's default
// nb = 32) on the offset-slot layout: k_big_resid_pat / k_big_sweep_pat's
// arithmetic with slot k of every row at column row + doff[k] -- coalesced
// value loads, no pattern-table reads.  One CTA per 256-row tile, a row per
// thread; the in-block sweeps gather w from global memory (other tiles).
// ---------------------------------------------------------------------------
template <typename T, bool FIRST>
__global__ void __launch_bounds__(kCtaThreads) k_big_dia_resid(const PassArgs<T> a, T *w0) {
  pdl_wait();  // (launched with programmatic dependent launch inside a solve: everything read below is the predecessor's)
  if (gated_off(a)) return;
  const TileDesc d = a.td[blockIdx.x];
  const int row = d.lo + threadIdx.x;
  if (row >= d.hi) return;
  const T rv = a.r64 != nullptr ? narrow_checked(a, a.r64[row], row, FIRST) : a.rT[row];
  const T *vb = a.dval + static_cast<long long>(row >> 5) * (32 * kDiaSlots) + (row & 31);
  T az = T(0);
  if (!FIRST) {
    const unsigned int m = __ldg(a.dmeta + row);
    const T *zr = a.zin + row;
    T v[kDiaSlots], g[kDiaSlots];
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++) {
      v[u] = __ldg(vb + 32 * u);
      g[u] = __ldg(zr + (((m >> u) & 1u) ? a.doff[u] : 0));  // (an absent slot's product is never added)
    }
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++)
      if ((m >> u) & 1u) az = add_rn(az, mul_rn(v[u], g[u]));
  }
  const T res = FIRST ? rv : sub_rn(rv, az);
  a.resbuf[row] = res;
  w0[row] = div_rn(res, __ldg(vb + 32 * kDiaDiag));
}

template <typename T, bool FIRST, bool LAST, bool FINISH>
__global__ void __launch_bounds__(kCtaThreads) k_big_dia_sweep(const PassArgs<T> a, const T *wsrc, T *wdst) {
  pdl_wait();
  if (gated_off(a)) return;
  __shared__ double ws[32];
  const int tile = blockIdx.x;
  const TileDesc d = a.td[tile];
  const int row = d.lo + threadIdx.x;
  double prod = 0.0;
  if (row < d.hi) {
    const unsigned int m = __ldg(a.dmeta + row) >> 8;  // in-block slots
    const T *vb = a.dval + static_cast<long long>(row >> 5) * (32 * kDiaSlots) + (row & 31);
    const T *wr = wsrc + row;
    T v[kDiaSlots], g[kDiaSlots];
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++) {
      v[u] = __ldg(vb + 32 * u);
      g[u] = wr[((m >> u) & 1u) ? a.doff[u] : 0];
    }
    T acc = T(0);
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++)
      if ((m >> u) & 1u) acc = add_rn(acc, mul_rn(v[u], g[u]));
    const T wn = add_rn(g[kDiaDiag], div_rn(sub_rn(a.resbuf[row], acc), v[kDiaDiag]));  // (the diagonal is in-block)
    if (!FINISH) {
      wdst[row] = wn;
    } else {
      const T zo = FIRST ? wn : add_rn(a.zin[row], wn);
      if (a.zout != nullptr) st_keep(a.zout + row, zo);
      if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
      if (LAST && a.part != nullptr) prod = __dmul_rn(a.r64[row], static_cast<double>(zo));
    }
  }
  if (FINISH && LAST && a.part != nullptr) {
    const double tot = block_tree<kTileThreads>(prod, ws);
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
    finish_grid(a.st, 0, kStepRho, ChunkCtx{a.st != nullptr ? a.csum : nullptr, a.part, a.g.ntiles, a.g.poll}, ws, true);
  }
}

// ---------------------------------------------------------------------------
// Whole solve in ONE persistent cooperative kernel, for problems of at most
// one tile per SM on the offset-slot layout (C1: 128 tiles).  Such a problem
// is L2-resident and each of the three kernels of an iteration is almost all
// fixed cost (launch, TMA round trip, grid ticket, final-CTA sum, drain):
// ~7 us per kernel against < 1 us of work.  Here CTA t owns tile t for the
// whole solve: its rows' x, r, p stay in registers, its matrix values (fp32
// and fp64 instance, operator) in shared memory; the three dependent global
// sums of an iteration are three grid barriers (release add + acquire spin on
// one counter), after which EVERY CTA sums the tile partials in the fixed
// order and runs the scalar step on its own copy of the solver state -- all
// copies stay identical, CTA 0 writes the trace.  Vectors other CTAs gather
// (pass outputs, z, p) go through global memory (L2: __ldcg).  Arithmetic,
// sum orders and the policy logic are those of the three-kernel iteration,
// so the solve is bit-identical to it (and to the oracle's device order).
// ---------------------------------------------------------------------------
struct SmallArgs {
  const float *dval32;    // offset-slot values: fp32 instance (null: uniform policy)
  const double *dval64;   // fp64 instance (null: fixed-low policy)
  const double *dvalop;   // the operator
  const uint16_t *dmeta;
  const TileDesc *td;
  int doff[8];
  int ntiles, k, t;
  double *x, *r;          // in: x0 and r0 = b - A x0; out: the solution (and final r)
  double *z;              // final z of the iteration, widened (gathered by the p rebuild)
  double *pA, *pB;        // search direction, alternating
  float *zA32, *zB32;     // pass outputs (fp32 instance)
  double *zA64, *zB64;    //              (fp64 instance)
  double *part_rz, *part_pq, *part_rr;
  unsigned int *bar;      // grid barrier counter (zero at launch)
  SolverState *st;
};

__device__ __forceinline__ void grid_bar(unsigned int *bar, unsigned int &target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// in-block sweeps of one row (w in, w out) against the tile's s_w
template <typename T>
__device__ __forceinline__ T small_sweeps(const SmallArgs &a, const T *v, unsigned int inb, int ti, bool valid,
                                          T res, T w, T *s_w) {
  s_w[ti] = w;
  for (int sw = 1; sw < a.t; sw++) {
    __syncthreads();
    T acc = T(0);
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++)
      if (valid && ((inb >> u) & 1u)) acc = add_rn(acc, mul_rn(v[32 * u], s_w[ti + a.doff[u]]));
    __syncthreads();
    w = add_rn(w, div_rn(sub_rn(res, acc), v[32 * kDiaDiag]));
    s_w[ti] = w;
  }
  __syncthreads();  // (s_w is rewritten by the next pass)
  return w;
}

// first pass z1 = D_b^{-1} r of the row (bjac_first_body's arithmetic), stored for the other tiles
template <typename T>
__device__ __forceinline__ T small_first(const SmallArgs &a, const T *v, unsigned int m, int ti, int row, bool valid,
                                         double ri, T *s_w, T *zout, T &rv) {
  rv = T(0);
  if (valid) {
    rv = narrow_or_copy<T>(ri);
    if (sizeof(T) == 4 && isinf(rv) && isfinite(ri)) {
      atomicAdd(&a.st->ovf_count, 1ull);
      atomicMin(&a.st->ovf_first, static_cast<long long>(row));
    }
  }
  T w = valid ? div_rn(rv, v[32 * kDiaDiag]) : T(0);
  w = small_sweeps<T>(a, v, m >> 8, ti, valid, rv, w, s_w);
  if (valid) zout[row] = w;
  return w;
}

// a pass after the first: z_out = z_in + D_b^{-1}(r - A z_in)
template <typename T>
__device__ __forceinline__ T small_pass(const SmallArgs &a, const T *v, unsigned int m, int ti, int row, bool valid,
                                        T rv, const T *zin, T *s_w) {
  T zown = T(0), res = T(0), w = T(0);
  if (valid) {
    T g[kDiaSlots];
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++) g[u] = __ldcg(zin + row + (((m >> u) & 1u) ? a.doff[u] : 0));
    T az = T(0);
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++)
      if ((m >> u) & 1u) az = add_rn(az, mul_rn(v[32 * u], g[u]));
    zown = g[kDiaDiag];
    res = sub_rn(rv, az);
    w = div_rn(res, v[32 * kDiaDiag]);
  }
  w = small_sweeps<T>(a, v, m >> 8, ti, valid, res, w, s_w);
  return add_rn(zown, w);
}

// the preconditioner of the iteration from its first pass on (z1 in zA): returns z widened
template <typename T>
__device__ __forceinline__ double small_rest(const SmallArgs &a, const T *v, unsigned int m, int ti, int row,
                                             bool valid, T rv, T z1, T *zA, T *zB, T *s_w, unsigned int &target,
                                             bool synced) {
  T z = z1;
  for (int pass = 1; pass < a.k; pass++) {
    // the previous pass's output of every tile must be stored (synced: z1 was, before the r.r barrier)
    if (pass > 1 || !synced) grid_bar(a.bar, target);
    const T *zin = (pass - 1) & 1 ? zB : zA;
    z = small_pass<T>(a, v, m, ti, row, valid, rv, zin, s_w);
    if (valid && pass + 1 < a.k) (pass & 1 ? zB : zA)[row] = z;
  }
  return static_cast<double>(z);
}

__global__ void __launch_bounds__(kCtaThreads) k_solve_small(const SmallArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(16) unsigned long long s_state[kStWords];
  __shared__ double ws[32];
  __shared__ float s_w32[kTileRows];
  __shared__ double s_w64[kTileRows];
  constexpr int kSlab = kTileRows * kDiaSlots;  // entries of a tile's value slab
  double *s_op = reinterpret_cast<double *>(smem);
  double *s_v64 = a.dval64 == nullptr ? nullptr : (a.dval64 == a.dvalop ? s_op : s_op + kSlab);
  float *s_v32 = reinterpret_cast<float *>(s_op + ((a.dval64 != nullptr && a.dval64 != a.dvalop) ? 2 : 1) * kSlab);
  const int tile = blockIdx.x, ti = threadIdx.x;
  const TileDesc d = a.td[tile];
  const int row = d.lo + ti;
  const bool valid = row < d.hi;
  SolverState *L = reinterpret_cast<SolverState *>(s_state);
  if (ti < kStWords) s_state[ti] = __ldcg(reinterpret_cast<const unsigned long long *>(a.st) + ti);
  {  // the tile's value slabs (rows past the tile: zero)
    const long long g0 = static_cast<long long>(kDiaSlots) * d.lo;
    const int cnt = kDiaSlots * (((d.hi - d.lo) + 31) & ~31);
    for (int i = ti; i < kSlab; i += kCtaThreads) {
      s_op[i] = i < cnt ? a.dvalop[g0 + i] : 0.0;
      if (s_v64 != nullptr && s_v64 != s_op) s_v64[i] = i < cnt ? a.dval64[g0 + i] : 0.0;
      if (a.dval32 != nullptr) s_v32[i] = i < cnt ? a.dval32[g0 + i] : 0.f;
    }
  }
  const unsigned int m = valid ? a.dmeta[row] : 0u;
  const int vo = (ti >> 5) * (32 * kDiaSlots) + (ti & 31);  // slot u of the row at vo + 32 u
  const double *vop = s_op + vo;
  const double *v64 = s_v64 != nullptr ? s_v64 + vo : nullptr;
  const float *v32 = s_v32 + vo;
  double xi = valid ? a.x[row] : 0.0, ri = valid ? a.r[row] : 0.0, pi = 0.0;
  unsigned int target = 0;
  int cur = 0;  // pold = cur ? pB : pA
  __syncthreads();
  const bool lead = blockIdx.x == 0;
  float rv32 = 0.f, z1_32 = 0.f;
  double rv64 = 0.0, z1_64 = 0.0;
  // the first iteration's first pass
  if (L->branch == 1) z1_32 = small_first<float>(a, v32, m, ti, row, valid, ri, s_w32, a.zA32, rv32);
  else z1_64 = small_first<double>(a, v64, m, ti, row, valid, ri, s_w64, a.zA64, rv64);
  bool synced = false;  // every tile's z1 is stored and a grid barrier has passed since
  for (;;) {
    // ---- z = M^{-1} r (remaining passes), rho = r.z --------------------------
    const double zi = L->branch == 1
                          ? small_rest<float>(a, v32, m, ti, row, valid, rv32, z1_32, a.zA32, a.zB32, s_w32, target, synced)
                          : small_rest<double>(a, v64, m, ti, row, valid, rv64, z1_64, a.zA64, a.zB64, s_w64, target, synced);
    if (valid) a.z[row] = zi;
    {
      const double tot = block_tree<kTileThreads>(valid ? __dmul_rn(ri, zi) : 0.0, ws);
      if (ti == 0) a.part_rz[tile] = tot;
    }
    grid_bar(a.bar, target);
    {
      const double rho = fin_sum<8, 1>(a.part_rz, a.ntiles, ws);
      if (ti == 0) {
        L->ovf_count = __ldcg(&a.st->ovf_count);
        L->ovf_first = __ldcg(&a.st->ovf_first);
        scalar_step_body(kStepRho, rho, L, lead);
      }
      __syncthreads();
    }
    if (L->done) break;
    // ---- p = z + beta p, q = A p, pq = p.q ------------------------------------
    const bool first = L->first != 0;
    const double beta = L->beta;
    const double *pold = cur ? a.pB : a.pA;
    double q = 0.0;
    if (valid) {
      double pv[kDiaSlots];
#pragma unroll
      for (int u = 0; u < kDiaSlots; u++) {
        const int c = row + (((m >> u) & 1u) ? a.doff[u] : 0);
        const double zv = __ldcg(a.z + c);
        pv[u] = first ? zv : __dadd_rn(zv, __dmul_rn(beta, __ldcg(pold + c)));
      }
#pragma unroll
      for (int u = 0; u < kDiaSlots; u++)
        if ((m >> u) & 1u) q = __dadd_rn(q, __dmul_rn(vop[32 * u], pv[u]));
      pi = pv[kDiaDiag];
      (cur ? a.pA : a.pB)[row] = pi;
    }
    cur ^= 1;
    {
      const double tot = block_tree<kTileThreads>(valid ? __dmul_rn(pi, q) : 0.0, ws);
      if (ti == 0) a.part_pq[tile] = tot;
    }
    grid_bar(a.bar, target);
    {
      const double pq = fin_sum<8, 1>(a.part_pq, a.ntiles, ws);
      if (ti == 0) scalar_step_body(kStepPq, pq, L, lead);
      __syncthreads();
    }
    if (L->done) break;
    // ---- x += alpha p, r -= alpha q, rr = r.r, the next first pass -------------
    const double alpha = L->alpha;
    if (valid) {
      xi = __dadd_rn(xi, __dmul_rn(alpha, pi));
      ri = __dsub_rn(ri, __dmul_rn(alpha, q));
    }
    {
      const double tot = block_tree<kTileThreads>(valid ? __dmul_rn(ri, ri) : 0.0, ws);
      if (ti == 0) a.part_rr[tile] = tot;
    }
    if (L->branch == 1) z1_32 = small_first<float>(a, v32, m, ti, row, valid, ri, s_w32, a.zA32, rv32);
    else z1_64 = small_first<double>(a, v64, m, ti, row, valid, ri, s_w64, a.zA64, rv64);
    grid_bar(a.bar, target);
    {
      const double rr = fin_sum<8, 1>(a.part_rr, a.ntiles, ws);
      if (ti == 0) scalar_step_body(kStepRrZ, rr, L, lead);
      __syncthreads();
    }
    if (L->done) break;
    synced = true;
    if (!L->z1_ok) {  // the aMP branch changed: the speculative first pass (and its narrowing count) is void
      synced = false;
      if (lead && ti == 0) {
        a.st->ovf_count = 0ull;
        a.st->ovf_first = 0x7fffffffffffffffLL;
      }
      grid_bar(a.bar, target);
      if (L->branch == 1) z1_32 = small_first<float>(a, v32, m, ti, row, valid, ri, s_w32, a.zA32, rv32);
      else z1_64 = small_first<double>(a, v64, m, ti, row, valid, ri, s_w64, a.zA64, rv64);
    }
  }
  if (valid) {
    a.x[row] = xi;
    a.r[row] = ri;
  }
  if (lead && ti < 32) {  // the final state (state_store's ranges; the narrowing counters stay as counted)
    if (ti == 0) {
      L->ovf_count = __ldcg(&a.st->ovf_count);
      L->ovf_first = __ldcg(&a.st->ovf_first);
    }
    __syncwarp();
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(a.st);
    constexpr int a1 = static_cast<int>(offsetof(SolverState, tr_relres) / 8);
    constexpr int b0 = static_cast<int>(offsetof(SolverState, dist) / 8), b1 = static_cast<int>(offsetof(SolverState, cond) / 8);
    for (int i = ti; i < a1 + (b1 - b0); i += 32) {
      const int wd = i < a1 ? i : b0 + (i - a1);
      dst[wd] = s_state[wd];
    }
  }
}

// Setup: per-row masks of the offset-slot layout from the row metadata
// (pattern id, in-block slot range) and pslot[pid * kSlots + j] = the
// offset slot of the pattern's j-th stored entry; any[0] collects the slots
// that are in-block somewhere.
__global__ void k_dia_meta(long long n, const uint16_t *meta, const int *pat, const signed char *pslot,
                           uint16_t *dmeta, unsigned int *any) {
  unsigned int seen = 0u;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const uint16_t m = meta[r];
    const int pid = meta_pid(m), len = pat_len(pat[pid * kPatStride]);
    unsigned int have = 0u, inb = 0u;
    for (int j = 0; j < len; j++) {
      const unsigned int bit = 1u << pslot[pid * kSlots + j];
      have |= bit;
      if (j >= meta_i0(m) && j < meta_i1(m)) inb |= bit;
    }
    dmeta[r] = static_cast<uint16_t>(have | (inb << 8));
    seen |= inb;
  }
  if (seen) atomicOr(any, seen);
}

// Setup: the near slots (kDiaDiag - 1 .. + 1) of the offset-slot values, 3 per row
template <typename E>
__global__ void k_dia_near(long long n, const E *dval, E *out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long src = (r >> 5) * (32 * kDiaSlots) + (r & 31), dst = (r >> 5) * (32 * kNearSlots) + (r & 31);
#pragma unroll
    for (int u = 0; u < kNearSlots; u++) out[dst + 32 * u] = dval[src + 32 * (kDiaDiag - 1 + u)];
  }
}

// Setup: SELL-32 values into the offset-slot layout (out zeroed before)
template <typename E>
__global__ void k_dia_pack(long long n, const int *sp, const E *sval, const uint16_t *meta, const int *pat,
                           const signed char *pslot, E *out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int pid = meta_pid(meta[r]), len = pat_len(pat[pid * kPatStride]);
    const long long src = sp[r >> 5] + (r & 31), dst = (r >> 5) * (32 * kDiaSlots) + (r & 31);
    for (int j = 0; j < len; j++) out[dst + 32 * pslot[pid * kSlots + j]] = sval[src + 32 * j];
  }
}

// ---------------------------------------------------------------------------
// Warp-per-tile fused BJAC pass.  Each consumer warp owns a whole tile, 8
// rows per lane (row lane + 32 k), so the inner sweeps need only __syncwarp
// (the tile's w lives in a warp-private shared array) and the tile's r.z
// sum is the same tree as include/mpbjac_order.h's (virtual warp k = rows
// 32k..32k+31 butterflied, then the 8 warp sums butterflied with +0 padding)
// without any CTA barrier.  Warps run their tiles independently, each with
// 8 rows x up to 7 z_in gathers of memory-level parallelism, where the CTA-
// wide version stalled all warps at every sweep barrier.  Consumer warp c
// takes ring stages c, c + W, c + 2W, ... (ns = W x depth stages); the
// producer ends the walk with one end marker per warp (ring_end).
// Plans with generic rows keep k_bjac_tile.
// ---------------------------------------------------------------------------
constexpr int kWtRows = kTileRows / 32;  // rows per lane
#ifndef MPB_WT_WARPS
#define MPB_WT_WARPS 4
#endif
constexpr int kWtWarps = MPB_WT_WARPS;   // consumer warps per CTA
constexpr int kWtMaxStages = 16;
constexpr int kWtBatch = 4;              // rows per lane whose gathers are in flight together

// tile sum of one value per row (prod[k] = row lane + 32 k) in the fixed
// order; the result is valid in every lane
__device__ __forceinline__ double wt_tile_sum(const double (&prod)[kWtRows]) {
  const int lane = threadIdx.x & 31;
  double r = 0.0;
#pragma unroll
  for (int k = 0; k < kWtRows; k++) {
    const double wsum = warp_bfly(prod[k]);
    if (lane == k) r = wsum;
  }
  return warp_bfly(r);
}

// One tile of a pass that reads the full rows (not the in-block-only first
// pass): z_out = z_in + D_b^{-1}(r - A z_in), the in-block sweeps in s_w.
template <typename T, bool FIRST, bool LAST, int KS>
__device__ __forceinline__ void wt_pass_tile(const PassArgs<T> &a, int tile, const TileDesc &d, const T *val,
                                             const int *spp, const uint16_t *mt, const double *r64t, const T *rTt,
                                             const int *s_pat, T *s_w) {
  const int lane = threadIdx.x & 31;
  T res[kWtRows], dd[kWtRows], w[kWtRows], zown[kWtRows];
#pragma unroll
  for (int kb = 0; kb < kWtRows; kb += kWtBatch) {
    T g[kWtBatch][KS], v[kWtBatch][KS];
    int len[kWtBatch];
#pragma unroll
    for (int q = 0; q < kWtBatch; q++) {  // issue every gather of the batch first
      const int k = kb + q, i = lane + 32 * k, row = d.lo + i;
      const bool valid = row < d.hi;
      const int ii = valid ? i : 0;
      const int *P = s_pat + meta_pid(mt[ii]) * kPatStride;
      const int base = spp[((d.lo + ii) >> 5) - d.s0] - d.e0 + ((d.lo + ii) & 31);
      len[q] = valid ? pat_len(P[0]) : 0;
      dd[k] = valid ? val[base + 32 * pat_dpos(P[0])] : T(1);
      const T *zr = FIRST ? nullptr : a.zin + d.lo + ii;
      if (!FIRST) zown[k] = __ldg(zr);
#pragma unroll
      for (int u = 0; u < KS; u++) {
        v[q][u] = u < len[q] ? val[base + 32 * u] : T(0);
        if (!FIRST) g[q][u] = __ldg(zr + P[1 + u]);  // offsets past len are 0
      }
    }
#pragma unroll
    for (int q = 0; q < kWtBatch; q++) {
      const int k = kb + q, i = lane + 32 * k, row = d.lo + i;
      if (row >= d.hi) {
        res[k] = T(0);
        w[k] = T(0);
        continue;
      }
      const T rv = r64t != nullptr ? narrow_checked(a, r64t[i], row, FIRST) : rTt[i];
      T az = T(0);
      if (!FIRST) {
#pragma unroll
        for (int u = 0; u < KS; u++)
          if (u < len[q]) az = add_rn(az, mul_rn(v[q][u], g[q][u]));
      }
      res[k] = FIRST ? rv : sub_rn(rv, az);
      w[k] = div_rn(res[k], dd[k]);
      s_w[i] = w[k];
    }
  }
  for (int s = 1; s < a.t; s++) {  // inner sweeps over the in-block entries
    __syncwarp();
    T acc[kWtRows];
#pragma unroll
    for (int k = 0; k < kWtRows; k++) {
      const int i = lane + 32 * k, row = d.lo + i;
      acc[k] = T(0);
      if (row >= d.hi) continue;
      const uint16_t m = mt[i];
      const int *P = s_pat + meta_pid(m) * kPatStride + 1;
      const int base = spp[(row >> 5) - d.s0] - d.e0 + (row & 31);
#pragma unroll 1
      for (int j = meta_i0(m); j < meta_i1(m); j++) acc[k] = add_rn(acc[k], mul_rn(val[base + 32 * j], s_w[i + P[j]]));
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kWtRows; k++) {
      const int i = lane + 32 * k;
      if (d.lo + i >= d.hi) continue;
      w[k] = add_rn(w[k], div_rn(sub_rn(res[k], acc[k]), dd[k]));
      s_w[i] = w[k];
    }
  }
  double prod[kWtRows];
#pragma unroll
  for (int k = 0; k < kWtRows; k++) {
    const int i = lane + 32 * k, row = d.lo + i;
    prod[k] = 0.0;
    if (row >= d.hi) continue;
    const T zo = FIRST ? w[k] : add_rn(zown[k], w[k]);
    if (a.zout != nullptr) st_keep(a.zout + row, zo);
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) prod[k] = __dmul_rn(r64t[i], static_cast<double>(zo));
  }
  if (LAST && a.part != nullptr) {
    const double tot = wt_tile_sum(prod);
    if (lane == 0) put_part(a.part + tile, tot);
  }
  __syncwarp();  // s_w is reused by the warp's next tile
}

// One tile of the in-block-only first pass (z1 = D_b^{-1} r): values and slice
// pointers of the plan's in-block SELL layout; res[k] = the row's residual.
template <typename T>
__device__ __forceinline__ void wt_first_tile(const PassArgs<T> &a, const TileDesc &d, const T *val, const int *spp,
                                              const uint16_t *mt, const T (&res)[kWtRows], const int *s_pat,
                                              T *s_w) {
  const int lane = threadIdx.x & 31;
  T dd[kWtRows], w[kWtRows];
#pragma unroll
  for (int k = 0; k < kWtRows; k++) {
    const int i = lane + 32 * k, row = d.lo + i;
    dd[k] = T(1);
    w[k] = T(0);
    if (row >= d.hi) continue;
    const uint16_t m = mt[i];
    const int *P = s_pat + meta_pid(m) * kPatStride;
    const int base = spp[(row >> 5) - d.s0] - d.ie0 + (row & 31);
    dd[k] = val[base + 32 * (pat_dpos(P[0]) - meta_i0(m))];
    w[k] = div_rn(res[k], dd[k]);
    s_w[i] = w[k];
  }
  for (int s = 1; s < a.t; s++) {
    __syncwarp();
    T acc[kWtRows];
#pragma unroll
    for (int k = 0; k < kWtRows; k++) {
      const int i = lane + 32 * k, row = d.lo + i;
      acc[k] = T(0);
      if (row >= d.hi) continue;
      const uint16_t m = mt[i];
      const int i0 = meta_i0(m), nib = meta_i1(m) - i0;
      const int *P = s_pat + meta_pid(m) * kPatStride + 1 + i0;
      const int base = spp[(row >> 5) - d.s0] - d.ie0 + (row & 31);
#pragma unroll 1
      for (int j = 0; j < nib; j++) acc[k] = add_rn(acc[k], mul_rn(val[base + 32 * j], s_w[i + P[j]]));
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kWtRows; k++) {
      const int i = lane + 32 * k;
      if (d.lo + i >= d.hi) continue;
      w[k] = add_rn(w[k], div_rn(sub_rn(res[k], acc[k]), dd[k]));
      s_w[i] = w[k];
    }
  }
#pragma unroll
  for (int k = 0; k < kWtRows; k++) {
    const int row = d.lo + lane + 32 * k;
    if (row >= d.hi) continue;
    if (a.zout != nullptr) st_keep(a.zout + row, w[k]);
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(w[k]);
  }
  __syncwarp();
}

template <typename T, bool FIRST, bool LAST, bool R64, int KS, bool TWO>
__global__ void __launch_bounds__(kWtWarps * 32 + 32) k_bjac_wt(const PassArgs<T> a) {
  constexpr int NC = kWtWarps * 32;
  constexpr int kFinRpt = NC >= kFinThreads ? 1 : kFinThreads / NC;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ RingT<kWtMaxStages> R;
  __shared__ T s_w[kWtWarps][kTileRows];
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  const int ns = a.g.ns;
  constexpr bool kIB = FIRST && !LAST;  // first pass alone: in-block entries only
  const StageLayout L = bjac_layout<T, FIRST, R64>(a.g);
  load_patterns(s_pat, a.pat, a.g.npat);
  ring_init(R, ns, 32);  // one consumer warp per stage
  if (threadIdx.x >= NC) {  // producer warp
    using RT = typename std::conditional<R64, double, T>::type;
    const RT *rsrc = R64 ? reinterpret_cast<const RT *>(a.r64) : reinterpret_cast<const RT *>(a.rT);
    const ChunkCtx ck{(TWO && LAST && a.part != nullptr && a.st != nullptr) ? a.csum : nullptr, a.part, a.g.ntiles,
                      TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      if (kIB)
        produce<T, RT, uint8_t, uint8_t, true>(R, st, a.td, tile, a.g, L, smem + st * L.bytes, a.ib_sp, a.ib_col,
                                               a.ib_val, a.meta, rsrc, nullptr, nullptr,
                                               static_cast<const uint8_t *>(nullptr), part);
      else
        produce<T, RT, uint8_t, uint8_t>(R, st, a.td, tile, a.g, L, smem + st * L.bytes, a.sp, a.scol, a.sval,
                                         a.meta, rsrc, nullptr, nullptr, static_cast<const uint8_t *>(nullptr), part);
    };
    auto gated = [&]() { return gated_off(a); };
    if (TWO && ck.csum != nullptr && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, kWtWarps, a.td);
    else if (threadIdx.x == NC)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, kWtWarps, a.td);
    else
      pdl_wait();
    if (gated_off(a)) return;
  } else {
    pdl_wait();
    if (gated_off(a)) return;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T *sw = s_w[c];
    int st = c, phase = 0;
    for (;;) {
      mbar_wait(&R.full[st], phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * L.bytes;
      const bool ok = R.ok[st] != 0;
      if (kIB) {
        const T *val = ok ? reinterpret_cast<const T *>(sb + L.val) : a.ib_val + d.ie0;
        const int *spp = ok ? staged(sb + L.sp, a.ib_sp, d.s0, d.s1 + 1) : a.ib_sp + d.s0;
        const uint16_t *mt = ok ? staged(sb + L.meta, a.meta, d.lo, d.hi) : a.meta + d.lo;
        T rv[kWtRows];
#pragma unroll
        for (int k = 0; k < kWtRows; k++) {
          const int i = lane + 32 * k, row = d.lo + i;
          rv[k] = T(0);
          if (row >= d.hi) continue;
          if (R64) rv[k] = narrow_checked(a, ok ? staged(sb + L.v0, a.r64, d.lo, d.hi)[i] : a.r64[row], row, true);
          else rv[k] = ok ? staged(sb + L.v0, a.rT, d.lo, d.hi)[i] : a.rT[row];
        }
        wt_first_tile<T>(a, d, val, spp, mt, rv, s_pat, sw);
      } else {
        const T *val = ok ? reinterpret_cast<const T *>(sb + L.val) : a.sval + d.e0;
        const int *spp = ok ? staged(sb + L.sp, a.sp, d.s0, d.s1 + 1) : a.sp + d.s0;
        const uint16_t *mt = ok ? staged(sb + L.meta, a.meta, d.lo, d.hi) : a.meta + d.lo;
        const double *r64t = R64 ? (ok ? staged(sb + L.v0, a.r64, d.lo, d.hi) : a.r64 + d.lo) : nullptr;
        const T *rTt = R64 ? nullptr : (ok ? staged(sb + L.v0, a.rT, d.lo, d.hi) : a.rT + d.lo);
        wt_pass_tile<T, FIRST, LAST, KS>(a, tile, d, val, spp, mt, r64t, rTt, s_pat, sw);
      }
      if (lane == 0) mbar_arrive(&R.empty[st]);
      st += kWtWarps;
      if (st >= ns) {
        st -= ns;
        phase ^= 1;
      }
    }
  }
  pdl_trigger();  // dependents may launch into the SMs this grid drains
  if (LAST && a.part != nullptr)
    finish_grid<16, kFinRpt>(a.st, 0, kStepRho, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---------------------------------------------------------------------------
// Flat (non-persistent) BJAC pass, no TMA ring: one CTA per tile, one row per
// thread, operands loaded straight from global memory (matrix values and
// row metadata before the grid dependency wait -- they do not depend on the
// previous kernel -- then the residual and the z_in gathers).  Many small
// resident CTAs (8 per SM) hide each other's load latency and barriers.
// Pattern rows only; one-level sums (<= MPB_ONE_LEVEL_TILES tiles).
// ---------------------------------------------------------------------------
template <typename T, bool FIRST, bool LAST, int KS>
__global__ void __launch_bounds__(kTileRows) k_bjac_flat(const PassArgs<T> a) {
  __shared__ T s_w[kTileRows];
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  const int tile = blockIdx.x;
  const TileDesc d = a.td[tile];
  const int i = threadIdx.x, row = d.lo + i;
  const bool valid = row < d.hi;
  const int rr = valid ? row : d.lo;
  const uint16_t m = __ldg(a.meta + rr);
  const int sb = __ldg(a.sp + (rr >> 5));
  const int width = (__ldg(a.sp + (rr >> 5) + 1) - sb) >> 5;
  const int base = sb + (rr & 31);
  T v[KS];
  const uint64_t pol = policy_evict_first();
#pragma unroll
  for (int u = 0; u < KS; u++) v[u] = u < width ? ld_stream(a.sval + base + 32 * u, pol) : T(0);
  load_patterns(s_pat, a.pat, a.g.npat);
  __syncthreads();
  pdl_wait();
  if (gated_off(a)) return;
  const int *P = s_pat + meta_pid(m) * kPatStride;
  const int hdr = P[0], len = pat_len(hdr);
  const T rv = narrow_checked(a, a.r64[rr], rr, FIRST);
  T az = T(0), zown = T(0);
  if (!FIRST) {
    const T *zr = a.zin + rr;
    zown = __ldg(zr);
    T g[KS];
#pragma unroll
    for (int u = 0; u < KS; u++) g[u] = __ldg(zr + P[1 + u]);
#pragma unroll
    for (int u = 0; u < KS; u++)
      if (u < len) az = add_rn(az, mul_rn(v[u], g[u]));
  }
  T dd = T(1);
#pragma unroll
  for (int u = 0; u < KS; u++)
    if (u == pat_dpos(hdr)) dd = v[u];
  const T res = FIRST ? rv : sub_rn(rv, az);
  T w = div_rn(res, dd);
  s_w[i] = w;
  const int i0 = meta_i0(m), i1 = meta_i1(m);
  for (int s = 1; s < a.t; s++) {
    __syncthreads();
    T acc = T(0);
#pragma unroll
    for (int u = 0; u < KS; u++)
      if (u >= i0 && u < i1) acc = add_rn(acc, mul_rn(v[u], s_w[i + P[1 + u]]));
    __syncthreads();
    w = add_rn(w, div_rn(sub_rn(res, acc), dd));
    s_w[i] = w;
  }
  double prod = 0.0;
  if (valid) {
    const T zo = FIRST ? w : add_rn(zown, w);
    if (a.zout != nullptr) st_keep(a.zout + row, zo);
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) prod = __dmul_rn(a.r64[row], static_cast<double>(zo));
  }
  if (LAST && a.part != nullptr) {
    const double tot = block_tree<kTileThreads>(prod, ws);
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
  }
  pdl_trigger();
  if (LAST && a.part != nullptr) finish_grid<16, 1>(a.st, 0, kStepRho, ChunkCtx{nullptr, a.part, a.g.ntiles, 0}, ws);
}

// ---- large blocks (> kTileRows rows): one launch per inner sweep ----------
// pass prologue: res = r - A z_in, d = diag, w0 = res / d
template <typename T, bool FIRST>
__global__ void __launch_bounds__(kCtaThreads) k_big_resid(const PassArgs<T> a, T *w0) {
  if (gated_off(a)) return;
  const TileDesc d = a.td[blockIdx.x];
  const int row = d.lo + threadIdx.x;
  if (row >= d.hi) return;
  const T rv = a.r64 != nullptr ? narrow_checked(a, a.r64[row], row, FIRST) : a.rT[row];
  const int s = row >> 5, sb = a.sp[s], width = (a.sp[s + 1] - sb) >> 5, base = sb + (row & 31);
  T az = T(0), dd = T(0);
  for (int j = 0; j < width; j++) {
    const int cj = __ldg(a.scol + base + 32 * j);
    if (cj < 0) continue;
    const T vj = __ldg(a.sval + base + 32 * j);
    if (!FIRST) az = add_rn(az, mul_rn(vj, __ldg(a.zin + cj)));
    if (cj == row) dd = vj;
  }
  const T res = FIRST ? rv : sub_rn(rv, az);
  a.resbuf[row] = res;
  a.dbuf[row] = dd;
  w0[row] = div_rn(res, dd);
}

// one inner sweep: w_new = w + (res - A_b w) / d  (A_b: in-block entries)
template <typename T>
__global__ void __launch_bounds__(kCtaThreads) k_big_sweep(const PassArgs<T> a, const T *wsrc, T *wdst) {
  if (gated_off(a)) return;
  const TileDesc d = a.td[blockIdx.x];
  const int row = d.lo + threadIdx.x;
  if (row >= d.hi) return;
  int blo, bhi;
  find_block_abs(a.boff + d.bf, d.nbk, row, blo, bhi);
  const int s = row >> 5, sb = a.sp[s], width = (a.sp[s + 1] - sb) >> 5, base = sb + (row & 31);
  T acc = T(0);
  for (int j = 0; j < width; j++) {
    const int cj = __ldg(a.scol + base + 32 * j);
    if (cj >= blo && cj < bhi) acc = add_rn(acc, mul_rn(__ldg(a.sval + base + 32 * j), wsrc[cj]));
  }
  wdst[row] = add_rn(wsrc[row], div_rn(sub_rn(a.resbuf[row], acc), a.dbuf[row]));
}

template <typename T, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kCtaThreads) k_big_finish(const PassArgs<T> a, const T *w) {
  if (gated_off(a)) return;
  __shared__ double ws[32];
  const int tile = blockIdx.x;
  const TileDesc d = a.td[tile];
  const int row = d.lo + threadIdx.x;
  double prod = 0.0;
  if (row < d.hi) {
    const T zo = FIRST ? w[row] : add_rn(a.zin[row], w[row]);
    if (a.zout != nullptr) st_keep(a.zout + row, zo);
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) prod = __dmul_rn(a.r64[row], static_cast<double>(zo));
  }
  if (LAST && a.part != nullptr) {
    const double tot = block_tree<kTileThreads>(prod, ws);
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
    // one CTA per tile (grid may exceed residency): the last CTA sums the chunks
    finish_grid(a.st, 0, kStepRho, ChunkCtx{a.st != nullptr ? a.csum : nullptr, a.part, a.g.ntiles, a.g.poll}, ws, true);
  }
}

// ---- large blocks, row-pattern versions (plans whose rows have patterns):
// the row's pattern gives its columns (row + offset, no column stream), its
// diagonal slot and -- through the plan's row metadata -- its in-block slot
// range [i0, i1), so no block search; the finish (z_out, r.z) is fused into
// the last inner sweep.  Generic rows (kMetaGeneric) take the column scans
// of k_big_resid / k_big_sweep in the same launch.
template <typename T, bool FIRST>
__global__ void __launch_bounds__(kCtaThreads) k_big_resid_pat(const PassArgs<T> a, T *w0) {
  if (gated_off(a)) return;
  const TileDesc d = a.td[blockIdx.x];
  const int row = d.lo + threadIdx.x;
  if (row >= d.hi) return;
  const T rv = a.r64 != nullptr ? narrow_checked(a, a.r64[row], row, FIRST) : a.rT[row];
  const int s = row >> 5, sb = __ldg(a.sp + s), base = sb + (row & 31);
  const uint16_t m = __ldg(a.meta + row);
  T az = T(0), dd = T(0);
  if (m != kMetaGeneric) {
    const int *P = a.pat + meta_pid(m) * kPatStride;
    const int hdr = __ldg(P), len = pat_len(hdr);
    dd = __ldg(a.sval + base + 32 * pat_dpos(hdr));
    if (!FIRST) {
      T v[kSlots], g[kSlots];
#pragma unroll
      for (int u = 0; u < kSlots; u++) {
        v[u] = u < len ? __ldg(a.sval + base + 32 * u) : T(0);
        g[u] = u < len ? __ldg(a.zin + row + __ldg(P + 1 + u)) : T(0);
      }
#pragma unroll
      for (int u = 0; u < kSlots; u++)
        if (u < len) az = add_rn(az, mul_rn(v[u], g[u]));
    }
  } else {
    const int width = (__ldg(a.sp + s + 1) - sb) >> 5;
    for (int j = 0; j < width; j++) {
      const int cj = __ldg(a.scol + base + 32 * j);
      if (cj < 0) continue;
      const T vj = __ldg(a.sval + base + 32 * j);
      if (!FIRST) az = add_rn(az, mul_rn(vj, __ldg(a.zin + cj)));
      if (cj == row) dd = vj;
    }
  }
  const T res = FIRST ? rv : sub_rn(rv, az);
  a.resbuf[row] = res;
  a.dbuf[row] = dd;
  w0[row] = div_rn(res, dd);
}

// one inner sweep w_new = w + (res - A_b w) / d; FINISH: the pass's last
// sweep also writes z_out = (z_in +) w_new and the r.z tile partial
template <typename T, bool FIRST, bool LAST, bool FINISH>
__global__ void __launch_bounds__(kCtaThreads) k_big_sweep_pat(const PassArgs<T> a, const T *wsrc, T *wdst) {
  if (gated_off(a)) return;
  __shared__ double ws[32];
  const int tile = blockIdx.x;
  const TileDesc d = a.td[tile];
  const int row = d.lo + threadIdx.x;
  double prod = 0.0;
  if (row < d.hi) {
    const int s = row >> 5, sb = __ldg(a.sp + s), base = sb + (row & 31);
    const uint16_t m = __ldg(a.meta + row);
    T acc = T(0);
    if (m != kMetaGeneric) {
      const int *P = a.pat + meta_pid(m) * kPatStride + 1;
      for (int j = meta_i0(m); j < meta_i1(m); j++)
        acc = add_rn(acc, mul_rn(__ldg(a.sval + base + 32 * j), wsrc[row + __ldg(P + j)]));
    } else {
      int blo, bhi;
      find_block_abs(a.boff + d.bf, d.nbk, row, blo, bhi);
      const int width = (__ldg(a.sp + s + 1) - sb) >> 5;
      for (int j = 0; j < width; j++) {
        const int cj = __ldg(a.scol + base + 32 * j);
        if (cj >= blo && cj < bhi) acc = add_rn(acc, mul_rn(__ldg(a.sval + base + 32 * j), wsrc[cj]));
      }
    }
    const T wn = add_rn(wsrc[row], div_rn(sub_rn(a.resbuf[row], acc), a.dbuf[row]));
    if (!FINISH) {
      wdst[row] = wn;
    } else {
      const T zo = FIRST ? wn : add_rn(a.zin[row], wn);
      if (a.zout != nullptr) st_keep(a.zout + row, zo);
      if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
      if (LAST && a.part != nullptr) prod = __dmul_rn(a.r64[row], static_cast<double>(zo));
    }
  }
  if (FINISH && LAST && a.part != nullptr) {
    const double tot = block_tree<kTileThreads>(prod, ws);
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
    finish_grid(a.st, 0, kStepRho, ChunkCtx{a.st != nullptr ? a.csum : nullptr, a.part, a.g.ntiles, a.g.poll}, ws, true);
  }
}

// ---------------------------------------------------------------------------
// p = z (first iteration) | z + beta * p_old   (solver.py:150-153)
// Streaming, persistent; z is the fp32 (low) or fp64 (high) branch output.
// ---------------------------------------------------------------------------
constexpr int kStreamTiles = 4;  // tiles per CTA iteration of the streaming kernels

__global__ void __launch_bounds__(kCtaThreads)
    k_pupdate(const TileDesc *td, int ntiles, const float *z32, const double *z64, double *p, const SolverState *st) {
  pdl_wait();
  if (st->done) return;
  const bool low = st->branch == 1;
  const bool first = st->first != 0;
  const double beta = st->beta;
  constexpr int U = kStreamTiles;
  for (int t0 = blockIdx.x; t0 < ntiles; t0 += U * gridDim.x) {
    int row[U];
    double zi[U], po[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int tile = t0 + u * gridDim.x;
      row[u] = -1;
      if (tile < ntiles) {
        const TileDesc d = td[tile];
        if (d.lo + (int)threadIdx.x < d.hi) row[u] = d.lo + threadIdx.x;
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      zi[u] = row[u] < 0 ? 0.0 : (low ? static_cast<double>(z32[row[u]]) : z64[row[u]]);
      po[u] = (row[u] < 0 || first) ? 0.0 : p[row[u]];
    }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (row[u] >= 0) p[row[u]] = first ? zi[u] : __dadd_rn(zi[u], __dmul_rn(beta, po[u]));
  }
}

// ---------------------------------------------------------------------------
// q = A p and the p.q partial (solver.py:154-159), fp64 SELL-32.  Values,
// slice pointers and row metadata are staged; p_j is gathered through L1.
// ---------------------------------------------------------------------------
struct SpmvArgs {
  const int *sp;
  const int *scol;
  const double *sval;
  const uint16_t *meta;
  const int *pat;
  const TileDesc *td;
  unsigned int *ctr;
  TileGeom g;
  const double *p;  // search direction (k_pupdate output), or ...
  // ... (pnew != null) p = z (first) | z + beta pold computed where it is
  // gathered (solver.py:150-153 fused into the SpMV); own rows stored to pnew
  const float *z32;
  const double *z64;
  const double *pold;
  double *pnew;
  double *q;
  double *part;
  SolverState *st;
  double *csum;        // chunk sums of the two-level p.q sum (ChunkCtx)
  int prefetch;     // see PassArgs::prefetch
  // symmetric offset-slot layout (k_spmv_sym): U + s n holds each row's value
  // at column offset d[s] >= 0 (d[0] = 0, 0 where absent); the value at
  // offset -d[s] is row (i - d[s])'s U_s entry (A symmetric, checked at build)
  // offset-slot layout of the operator (k_spmv_dia; PassArgs::dval's layout in fp64)
  const double *dval;
  const uint16_t *dmeta;
  int doff[8];
  const double *U;
  const uint16_t *pmask;  // per row pattern: bit j = signed offset j (ascending) present
  int n;
  int S;
  int d[8];
};

// p_j as the SpMV reads it: stored (ZT = void) or rebuilt from z (ZT = the
// preconditioner branch's type) and the previous p -- every thread that
// needs p_j computes the same two roundings, so all copies agree bit for bit
template <typename ZT>
__device__ __forceinline__ double p_at(const SpmvArgs &a, int c, bool first, double beta) {
  if constexpr (std::is_same<ZT, void>::value) {
    return __ldg(a.p + c);
  } else {
    const double zv = std::is_same<ZT, float>::value ? static_cast<double>(__ldg(a.z32 + c)) : __ldg(a.z64 + c);
    return first ? zv : __dadd_rn(zv, __dmul_rn(beta, __ldg(a.pold + c)));
  }
}

template <int KS, typename ZT, bool GEN>
__device__ __forceinline__ void spmv_tile_body(const SpmvArgs &a, int tile, const TileDesc &d, const int *col,
                                               const double *val, const int *spp, const uint16_t *mt,
                                               const int *s_pat, double *ws, bool first, double beta) {
  double prod[kRowsPerThread];
#pragma unroll
  for (int k = 0; k < kRowsPerThread; k++) {
    const int tid = threadIdx.x + k * kConsumers, row = d.lo + tid;
    prod[k] = 0.0;
    if (row >= d.hi) continue;
    const int si = (row >> 5) - d.s0;
    const int sb = spp[si];
    const int base = sb - d.e0 + (row & 31);
    const uint16_t m = mt[tid];
    double acc = 0.0;
    if (!GEN || m != kMetaGeneric) {
      const int *P = s_pat + meta_pid(m) * kPatStride;
      const int len = pat_len(P[0]);
      double vv[KS], pv[KS];
#pragma unroll
      for (int u = 0; u < KS; u++) {
        vv[u] = u < len ? val[base + 32 * u] : 0.0;
        pv[u] = p_at<ZT>(a, row + P[1 + u], first, beta);
      }
#pragma unroll
      for (int u = 0; u < KS; u++)
        if (u < len) acc = __dadd_rn(acc, __dmul_rn(vv[u], pv[u]));
    } else {
      const int width = (spp[si + 1] - sb) >> 5;
      for (int j = 0; j < width; j++) {
        const int c = col[base + 32 * j];
        if (c >= 0) acc = __dadd_rn(acc, __dmul_rn(val[base + 32 * j], p_at<ZT>(a, c, first, beta)));
      }
    }
    a.q[row] = acc;
    const double pown = p_at<ZT>(a, row, first, beta);
    if (!std::is_same<ZT, void>::value) st_keep(a.pnew + row, pown);
    prod[k] = __dmul_rn(pown, acc);
  }
  const double tot = tile_tree_rows(prod, ws, kBarConsumers);
  if (threadIdx.x == 0) put_part(a.part + tile, tot);
}

__host__ __device__ inline StageLayout spmv_layout(const TileGeom &g) {
  return stage_layout(g.cap_e, 8, g.max_sl, g.cols != 0, true, 0, 0, 0);
}

// one tile of the SpMV with p stored or rebuilt (branch of the iteration)
template <int KS, bool GEN>
__device__ __forceinline__ void spmv_tile(const SpmvArgs &a, int tile, const TileDesc &d, const int *col,
                                          const double *val, const int *spp, const uint16_t *mt, const int *s_pat,
                                          double *ws, int mode, bool first, double beta) {
  if (mode == 0) spmv_tile_body<KS, void, GEN>(a, tile, d, col, val, spp, mt, s_pat, ws, first, beta);
  else if (mode == 1) spmv_tile_body<KS, float, GEN>(a, tile, d, col, val, spp, mt, s_pat, ws, first, beta);
  else spmv_tile_body<KS, double, GEN>(a, tile, d, col, val, spp, mt, s_pat, ws, first, beta);
}

template <int KS, bool GEN, bool TWO = false>
__global__ void MPB_WS_BOUNDS_SPMV k_spmv_pq(const SpmvArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  const int ns = a.g.ns;
  const StageLayout L = spmv_layout(a.g);
  load_patterns(s_pat, a.pat, a.g.npat);
  ring_init(R, ns);
  if (threadIdx.x >= kConsumers) {
    const ChunkCtx ck{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      produce<double, uint8_t, uint8_t, uint8_t, false, uint8_t>(R, st, a.td, tile, a.g, L, smem + st * L.bytes, a.sp,
                                                                 a.scol, a.sval, a.meta, nullptr, nullptr, nullptr,
                                                                 nullptr, part);
    };
    auto gated = [&]() { return a.st->done != 0; };
    if (TWO && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == kConsumers)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td);
    else
      pdl_wait();
    if (a.st->done) return;
  } else {
    pdl_wait();
    if (a.st->done) return;
    if (threadIdx.x == 0) tl_mark(a.st, 1, 0, false);
    const int mode = a.pnew == nullptr ? 0 : (a.st->branch == 1 ? 1 : 2);
    const bool first = a.st->first != 0;
    const double beta = a.st->beta;
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * L.bytes;
      if (R.ok[st]) {
        const int *col = (a.g.cols && d.ngen > 0) ? reinterpret_cast<const int *>(sb + L.col) : a.scol + d.e0;
        spmv_tile<KS, GEN>(a, tile, d, col, reinterpret_cast<const double *>(sb + L.val),
                      staged(sb + L.sp, a.sp, d.s0, d.s1 + 1), staged(sb + L.meta, a.meta, d.lo, d.hi), s_pat, ws,
                      mode, first, beta);
      } else {
        spmv_tile<KS, GEN>(a, tile, d, a.scol + d.e0, a.sval + d.e0, a.sp + d.s0, a.meta + d.lo, s_pat, ws, mode, first,
                      beta);
      }
      ring_release(R, st);
    }
    if (threadIdx.x == 0) tl_mark(a.st, 1, 1, true);
  }
  pdl_trigger();
  finish_grid<16, kFinRptWs>(a.st, 1, kStepPq, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---- SpMV on the offset-slot layout ------------------------------------------
// q = A p with p rebuilt where it is gathered (k_spmv_pq's arithmetic) on the
// offset-slot values of the operator: slot k of a row at a fixed shared-memory
// offset, column row + doff[k], the row's own p from the diagonal slot's
// gather.  One row per thread, 8 consumer warps that never meet at a CTA
// barrier: the tile's p.q sum is finished by the warp that arrives last on
// the stage's counter (the order of include/mpbjac_order.h).
constexpr uint32_t kDiaSpmvStage = kTileRows * kDiaSlots * 8u + kTileRows * 2u;

template <typename ZT>
__device__ __forceinline__ void dia_spmv_tile(const SpmvArgs &a, int tile, int lo, int nrows, const double *val,
                                              const uint16_t *dm, double *wsum, unsigned int *wcnt, bool first,
                                              double beta) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ti = threadIdx.x;
  double prod = 0.0;
  if (32 * warp < nrows) {  // warp-uniform (tiles hold a multiple of 64 rows)
    const int row = lo + ti;
    const unsigned int m = dm[ti];
    const double *vb = val + warp * (32 * kDiaSlots) + lane;
    double v[kDiaSlots], pv[kDiaSlots];
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++) {
      v[u] = vb[32 * u];
      // (an absent slot gathers the row's own p: its product is never added)
      pv[u] = p_at<ZT>(a, row + (((m >> u) & 1u) ? a.doff[u] : 0), first, beta);
    }
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < kDiaSlots; u++)
      if ((m >> u) & 1u) acc = __dadd_rn(acc, __dmul_rn(v[u], pv[u]));
    a.q[row] = acc;
    const double pown = pv[kDiaDiag];
    if (!std::is_same<ZT, void>::value) st_keep(a.pnew + row, pown);
    prod = __dmul_rn(pown, acc);
  }
  prod = warp_bfly(prod);
  if (lane == 0) wsum[warp] = prod;
  __syncwarp();
  unsigned int old = 0;
  if (lane == 0)
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(wcnt)) : "memory");
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old == kTileThreads / 32 - 1) {  // the tile's last warp: every warp sum is stored
    double t = lane < kTileThreads / 32 ? wsum[lane] : 0.0;
    t = warp_bfly(t);
    if (lane == 0) {
      *wcnt = 0u;
      put_part(a.part + tile, t);
    }
  }
}

template <bool TWO>
__global__ void __launch_bounds__(kWsThreads, 4) k_spmv_dia(const SpmvArgs a) {
  static_assert(kConsumers == kTileThreads, "one row per consumer thread");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ double ws[32];
  __shared__ double s_wsum[kMaxStages * (kTileThreads / 32)];
  __shared__ unsigned int s_wcnt[kMaxStages];
  if (threadIdx.x < kMaxStages) s_wcnt[threadIdx.x] = 0u;  // (published by ring_init's barrier)
  const int ns = a.g.ns;
  ring_init(R, ns);
  const bool red = a.g.red != 0;
  if (red && blockIdx.x == 0) {  // this CTA takes no tiles: its first warp streams the p.q sum
    pdl_wait();
    if (!a.st->done && threadIdx.x < 32) reduce_stream(a.st, kStepPq, a.part, a.g.ntiles);
    pdl_trigger();
    return;
  }
  if (threadIdx.x >= kConsumers) {
    const ChunkCtx ck{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0};
    // every staged byte is static (values, masks): all of it may stream
    // before the grid dependency wait; the dynamic part only arrives
    auto fill = [&](int st, int tile, int part) {
      if (part != kFillDynamic) {
        const TileDesc d = a.td[tile];
        R.desc[st] = d;
        R.ok[st] = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t rows = static_cast<uint32_t>(d.hi - d.lo);  // a multiple of 64
        unsigned char *stage = smem + st * kDiaSpmvStage;
        if (part == kFillAll) mbar_arrive_expect_tx(&R.full[st], rows * (kDiaSlots * 8u + 2u));
        else mbar_expect_tx(&R.full[st], rows * (kDiaSlots * 8u + 2u));
        bulk_g2s_stream(stage, a.dval + static_cast<long long>(kDiaSlots) * d.lo, rows * kDiaSlots * 8u, &R.full[st]);
        bulk_g2s(stage + kTileRows * kDiaSlots * 8u, a.dmeta + d.lo, rows * 2u, &R.full[st]);
      } else {
        mbar_arrive(&R.full[st]);
      }
    };
    auto gated = [&]() { return a.st->done != 0; };
    if (TWO && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == kConsumers)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td, gridDim.x - (red ? 1u : 0u));
    else
      pdl_wait();
    if (a.st->done) return;
  } else {
    pdl_wait();
    if (a.st->done) return;
    if (threadIdx.x == 0) tl_mark(a.st, 1, 0, false);
    const int mode = a.pnew == nullptr ? 0 : (a.st->branch == 1 ? 1 : 2);
    const bool first = a.st->first != 0;
    const double beta = a.st->beta;
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const int lo = R.desc[st].lo, nrows = R.desc[st].hi - lo;
      const unsigned char *sb = smem + st * kDiaSpmvStage;
      const double *val = reinterpret_cast<const double *>(sb);
      const uint16_t *dm = reinterpret_cast<const uint16_t *>(sb + kTileRows * kDiaSlots * 8u);
      double *wsum = s_wsum + st * (kTileThreads / 32);
      if (mode == 0) dia_spmv_tile<void>(a, tile, lo, nrows, val, dm, wsum, s_wcnt + st, first, beta);
      else if (mode == 1) dia_spmv_tile<float>(a, tile, lo, nrows, val, dm, wsum, s_wcnt + st, first, beta);
      else dia_spmv_tile<double>(a, tile, lo, nrows, val, dm, wsum, s_wcnt + st, first, beta);
      ring_release(R, st);
    }
    if (threadIdx.x == 0) tl_mark(a.st, 1, 1, true);
  }
  pdl_trigger();
  if (!red) finish_grid<16, kFinRptWs>(a.st, 1, kStepPq, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---- SpMV on the symmetric offset-slot layout --------------------------------
// A symmetric pattern-row matrix whose distinct column offsets are
// {-d[S-1] .. -d[1], 0, d[1] .. d[S-1]} stores only the S nonnegative-offset
// values of each row (U_s, slot-major): the stage carries the tile's U rows
// and its row metadata, and row i takes its lower entries (offset -d[s]) from
// row i - d[s]'s U_s through global memory (L2: those rows were streamed a
// few tiles earlier).  Ascending column order and one rounding per product
// and per add, as the SELL kernel: bit-identical.  8 (S = 4) or 12 bytes of
// values per row less than the SELL layout's 7 (9) slots.
constexpr int kSymMax = 6;

// Stage regions: U_0 rows [lo, hi); for s >= 1 with d[s] < kTileRows one
// window [lo - d[s], hi) (upper and lower entries), else two: [lo, hi) and
// the mirror rows [lo - d[s], hi - d[s]) -- every value the tile's rows use
// comes from shared memory.  Windows start clamped at row 0.
struct SymLayout {
  uint32_t meta, up[kSymMax], lo[kSymMax], bytes;  // lo[s] == up[s] for merged windows
};
__host__ __device__ inline uint32_t sym_win_bytes(int rows) {
  return al16u(static_cast<uint32_t>(rows) * 8u + 32u);
}
__host__ __device__ inline SymLayout spmv_sym_layout(int S, const int *d) {
  SymLayout L{};
  uint32_t off = 0;
  L.meta = off;
  off += al16u(static_cast<uint32_t>(kTileRows) * 2u + 16u);
  for (int s = 0; s < S; s++) {
    if (s == 0) {
      L.up[0] = L.lo[0] = off;
      off += sym_win_bytes(kTileRows);
    } else if (d[s] < kTileRows) {
      L.up[s] = L.lo[s] = off;
      off += sym_win_bytes(kTileRows + d[s]);
    } else {
      L.up[s] = off;
      off += sym_win_bytes(kTileRows);
      L.lo[s] = off;
      off += sym_win_bytes(kTileRows);
    }
  }
  L.bytes = off;
  return L;
}
// the window rows of slot s's lower region [a, b) and upper region [c, e)
__device__ __forceinline__ void sym_rows(const TileDesc &d, int ds, int s, int &a, int &b, int &c, int &e) {
  c = d.lo;
  e = d.hi;
  if (s == 0) {
    a = c;
    b = e;
  } else if (ds < kTileRows) {
    a = max(d.lo - ds, 0);
    b = d.hi;
  } else {
    a = max(d.lo - ds, 0);
    b = max(d.hi - ds, 0);
  }
}

__device__ __forceinline__ int mask_of(const uint16_t *s_mask, uint16_t m) { return s_mask[meta_pid(m)]; }

// soff[s]: byte offset (from the stage base) of the tile's row lo - d[s] + tid
// in slot s's lower window, soff[S + s] of row lo + tid in its upper window
// (the producer computes them per stage: one shared-memory read per slot here)
template <int S, typename ZT>
__device__ __forceinline__ void spmv_sym_tile_body(const SpmvArgs &a, int tile, const TileDesc &d,
                                                   const unsigned char *sb, const SymLayout &L, const int *soff,
                                                   const uint16_t *s_mask, double *ws, bool first, double beta) {
  const int tid = threadIdx.x, row = d.lo + tid;
  double prod[1] = {0.0};
  if (row < d.hi) {
    const uint16_t *mt = staged(sb + L.meta, a.meta, d.lo, d.hi);
    const int m = mask_of(s_mask, mt[tid]);
    const unsigned char *sbt = sb + tid * 8;
    double acc = 0.0;
#pragma unroll
    for (int s = S - 1; s >= 1; s--) {  // lower entries, most negative offset first
      if ((m >> (S - 1 - s)) & 1) {
        const int c = row - a.d[s];
        acc = __dadd_rn(acc, __dmul_rn(*reinterpret_cast<const double *>(sbt + soff[s]), p_at<ZT>(a, c, first, beta)));
      }
    }
    const double pown = p_at<ZT>(a, row, first, beta);
    acc = __dadd_rn(acc, __dmul_rn(*reinterpret_cast<const double *>(sbt + soff[S]), pown));  // diagonal
#pragma unroll
    for (int s = 1; s < S; s++) {
      if ((m >> (S - 1 + s)) & 1)
        acc = __dadd_rn(acc, __dmul_rn(*reinterpret_cast<const double *>(sbt + soff[S + s]),
                                       p_at<ZT>(a, row + a.d[s], first, beta)));
    }
    a.q[row] = acc;
    if (!std::is_same<ZT, void>::value) st_keep(a.pnew + row, pown);
    prod[0] = __dmul_rn(pown, acc);
  }
  const double tot = tile_tree_rows<double, 1>(prod, ws, kBarConsumers);
  if (threadIdx.x == 0) put_part(a.part + tile, tot);
}

template <int S, bool TWO = false>
__global__ void MPB_WS_BOUNDS_SPMV k_spmv_sym(const SpmvArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ double ws[32];
  __shared__ uint16_t s_mask[kPatMax];
  __shared__ int s_soff[kMaxStages][2 * kSymMax];
  const int ns = a.g.ns;
  const SymLayout L = spmv_sym_layout(S, a.d);
  for (int i = threadIdx.x; i < a.g.npat; i += blockDim.x) s_mask[i] = __ldg(a.pmask + i);
  ring_init(R, ns);
  if (threadIdx.x >= kConsumers) {
    const ChunkCtx ck{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0};
    // every staged byte is static (U, row metadata): all of it may stream
    // before the grid dependency wait; the dynamic part only arrives
    auto fill = [&](int st, int tile, int part) {
      unsigned char *stage = smem + st * L.bytes;
      if (part != kFillDynamic) {
        const TileDesc d = a.td[tile];
        R.desc[st] = d;
        R.ok[st] = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        uint32_t bytes = window_bytes(a.meta, d.lo, d.hi);
        for (int s = 0; s < S; s++) {
          const double *us = a.U + static_cast<long long>(s) * a.n;
          int wa, wb, wc, we;
          sym_rows(d, a.d[s], s, wa, wb, wc, we);
          if (wb > wa) bytes += window_bytes(us, wa, wb);
          if (s > 0 && a.d[s] >= kTileRows) bytes += window_bytes(us, wc, we);
        }
        if (part == kFillAll) mbar_arrive_expect_tx(&R.full[st], bytes);
        else mbar_expect_tx(&R.full[st], bytes);
        tma_window(stage + L.meta, a.meta, d.lo, d.hi, &R.full[st], true);
        for (int s = 0; s < S; s++) {
          const double *us = a.U + static_cast<long long>(s) * a.n;
          int wa, wb, wc, we;
          sym_rows(d, a.d[s], s, wa, wb, wc, we);
          if (wb > wa) tma_window(stage + L.lo[s], us, wa, wb, &R.full[st]);
          if (s > 0 && a.d[s] >= kTileRows) tma_window(stage + L.up[s], us, wc, we, &R.full[st]);
          // byte offsets of row (lo - d[s]) and row lo in the windows (may
          // point before a clamped window start: those rows are never read)
          const int skew_lo = static_cast<int>(window_of(us, wa, wb).skew);
          s_soff[st][s] = static_cast<int>(L.lo[s]) + skew_lo + 8 * (d.lo - a.d[s] - wa);
          if (s == 0 || a.d[s] < kTileRows) s_soff[st][S + s] = static_cast<int>(L.lo[s]) + skew_lo + 8 * (d.lo - wa);
          else s_soff[st][S + s] = static_cast<int>(L.up[s]) + static_cast<int>(window_of(us, wc, we).skew);
        }
      } else {
        mbar_arrive(&R.full[st]);
      }
    };
    auto gated = [&]() { return a.st->done != 0; };
    if (TWO && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == kConsumers)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td);
    else
      pdl_wait();
    if (a.st->done) return;
  } else {
    pdl_wait();
    if (a.st->done) return;
    const int mode = a.pnew == nullptr ? 0 : (a.st->branch == 1 ? 1 : 2);
    const bool first = a.st->first != 0;
    const double beta = a.st->beta;
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * L.bytes;
      const int *soff = s_soff[st];
      if (mode == 0) spmv_sym_tile_body<S, void>(a, tile, d, sb, L, soff, s_mask, ws, first, beta);
      else if (mode == 1) spmv_sym_tile_body<S, float>(a, tile, d, sb, L, soff, s_mask, ws, first, beta);
      else spmv_sym_tile_body<S, double>(a, tile, d, sb, L, soff, s_mask, ws, first, beta);
      ring_release(R, st);
    }
  }
  pdl_trigger();
  finish_grid<16, kFinRptWs>(a.st, 1, kStepPq, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// Symmetry check of pattern rows against the offset set d (S entries >= 0):
// counts entries (row i, offset o > 0) whose value differs bitwise from row
// i + o's value at offset -o, or whose mirror entry is missing.
__global__ void k_sym_check(long long n, const int *sp, const double *sval, const uint16_t *meta, const int *pat,
                            unsigned long long *bad) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(r);
    const uint16_t m = meta[row];
    if (m == kMetaGeneric) {
      atomicAdd(bad, 1ull);
      continue;
    }
    const int *P = pat + meta_pid(m) * kPatStride;
    const int len = pat_len(P[0]);
    const int base = sp[row >> 5] + (row & 31);
    for (int u = 0; u < len; u++) {
      const int o = P[1 + u];
      if (o == 0) continue;
      const int c = row + o;
      const uint16_t mc = meta[c];
      bool found = false;
      if (mc != kMetaGeneric) {
        const int *Q = pat + meta_pid(mc) * kPatStride;
        const int lc = pat_len(Q[0]);
        const int bc = sp[c >> 5] + (c & 31);
        for (int v = 0; v < lc; v++)
          if (Q[1 + v] == -o) {
            found = __double_as_longlong(sval[bc + 32 * v]) == __double_as_longlong(sval[base + 32 * u]);
            break;
          }
      }
      if (!found) atomicAdd(bad, 1ull);
    }
  }
}

// U_s[i] = row i's value at offset d[s] (0 where absent)
__global__ void k_sym_build(long long n, const int *sp, const double *sval, const uint16_t *meta, const int *pat,
                            int S, SpmvArgs da, double *U) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(r);
    const uint16_t m = meta[row];
    for (int s = 0; s < S; s++) U[s * n + r] = 0.0;
    if (m == kMetaGeneric) continue;
    const int *P = pat + meta_pid(m) * kPatStride;
    const int len = pat_len(P[0]);
    const int base = sp[row >> 5] + (row & 31);
    for (int u = 0; u < len; u++) {
      const int o = P[1 + u];
      if (o < 0) continue;
      for (int s = 0; s < S; s++)
        if (da.d[s] == o) U[s * n + r] = sval[base + 32 * u];
    }
  }
}

// x += alpha p ; r -= alpha q ; r.r partial   (solver.py:160-165)
// Persistent; each CTA iteration streams kStreamTiles tiles with every load
// issued up front and one barrier pair for their tile sums.
__global__ void __launch_bounds__(kCtaThreads)
    k_update(const TileDesc *td, int ntiles, double *x, const double *p, const double *q, double *r, double *part,
             SolverState *st, double *csum, int poll) {
  pdl_wait();
  if (st->done) return;
  __shared__ double ws[kStreamTiles][32];
  __shared__ double wsf[32];
  const double alpha = st->alpha;
  constexpr int U = kStreamTiles;
  for (int t0 = blockIdx.x; t0 < ntiles; t0 += U * gridDim.x) {
    int row[U];
    double xv[U], pv[U], qv[U], rv[U], sq[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int tile = t0 + u * gridDim.x;
      row[u] = -1;
      if (tile < ntiles) {
        const TileDesc d = td[tile];
        if (d.lo + (int)threadIdx.x < d.hi) row[u] = d.lo + threadIdx.x;
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool ok = row[u] >= 0;
      xv[u] = ok ? x[row[u]] : 0.0;
      pv[u] = ok ? p[row[u]] : 0.0;
      qv[u] = ok ? q[row[u]] : 0.0;
      rv[u] = ok ? r[row[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      sq[u] = 0.0;
      if (row[u] >= 0) {
        x[row[u]] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));
        const double rnew = __dsub_rn(rv[u], __dmul_rn(alpha, qv[u]));
        r[row[u]] = rnew;
        sq[u] = __dmul_rn(rnew, rnew);
      }
    }
    // lane j of a tile owns row j only (<= kTileThreads rows), so the tile
    // sum is the block tree of the per-row squares
    block_tree_multi<U>(sq, ws);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int tile = t0 + u * gridDim.x;
        if (tile < ntiles) put_part(part + tile, sq[u]);
      }
    }
  }
  pdl_trigger();
  const ChunkCtx ck{csum, part, ntiles, poll};
  chunk_duties_strided(ck, blockIdx.x, gridDim.x);
  finish_grid(st, 2, kStepRr, ck, wsf);
}

// Fused x/r update + the next iteration's first BJAC pass (solver.py:160-165
// then bjac.py:134-136 for the branch in force): each tile updates its own
// x and r rows, adds its r.r partial, narrows the new r (fp32 branch, with
// the overflow count) and runs the in-block sweeps into z1.  The last CTA
// runs kStepRrZ; if the step changes the branch, z1 is discarded and the
// standalone first pass of the new branch runs instead (z1_gate).
// MPB_UF_DIRECT=1 (experiment): x and q are read by the consumers straight
// from global memory instead of being staged (two bulk copies fewer per stage)
#ifndef MPB_UF_DIRECT
#define MPB_UF_DIRECT 0
#endif
constexpr bool kUfDirect = MPB_UF_DIRECT != 0;
template <typename T>
__host__ __device__ inline StageLayout update_first_layout(const TileGeom &g) {
  // v0 r, v1 x, v2 p, v3 q (fp64 slices)
  return stage_layout(g.cap_e, sizeof(T), g.max_sl, g.cols != 0, true, 8, kUfDirect ? 0 : 8, 8, kUfDirect ? 0 : 8);
}

// Staged tile of the fused update with a multiple of 32 rows at a 32-row-
// aligned start, pattern rows only (update_first_body's arithmetic without
// per-row validity branches; the in-block sweep unrolled to KI entries).
template <typename T, int KI>
__device__ __forceinline__ void update_first_full(const PassArgs<T> &a, int tile, const TileDesc &d, double alpha,
                                                  double *x, double *r, const double *xs, const double *ps,
                                                  const double *qs, const double *rs, const T *val, const int *spp,
                                                  const uint16_t *mt, const int *s_pat, T *s_w, double *ws) {
  const int tid = threadIdx.x, row = d.lo + tid;
  const bool valid = row < d.hi;  // warp-uniform
  const int ti = valid ? tid : 0;
  double sq = 0.0;
  T rv = T(0);
  if (valid) {
    st_evict_first(x + row, __dadd_rn(xs[ti], __dmul_rn(alpha, ps[ti])));  // (read again by the next update only)
    const double rn = __dsub_rn(rs[ti], __dmul_rn(alpha, qs[ti]));
    r[row] = rn;
    sq = __dmul_rn(rn, rn);
    rv = narrow_checked(a, rn, row, true);
  }
  const uint16_t m = mt[ti];
  const int i0 = meta_i0(m), nib = meta_i1(m) - i0;
  const int *P = s_pat + meta_pid(m) * kPatStride;
  const int base = spp[ti >> 5] - d.ie0 + (ti & 31);
  const T dd = val[base + 32 * (pat_dpos(P[0]) - i0)];
  P += 1 + i0;
  T w = div_rn(rv, dd);
  {
    double v[1] = {sq};
    const double tot = tile_tree_rows<double, 1>(v, ws, kBarConsumers);  // (its barriers also order s_w)
    if (threadIdx.x == 0) put_part(a.part + tile, tot);
  }
  s_w[tid] = w;
  for (int s = 1; s < a.t; s++) {
    named_sync(kBarConsumers, kTileThreads);
    T acc = T(0);
#pragma unroll
    for (int j = 0; j < KI; j++)
      if (j < nib) acc = add_rn(acc, mul_rn(val[base + 32 * j], s_w[tid + P[j]]));
    named_sync(kBarConsumers, kTileThreads);
    w = add_rn(w, div_rn(sub_rn(rv, acc), dd));
    s_w[tid] = w;
  }
  if (valid && a.zout != nullptr) st_keep(a.zout + row, w);
  if (valid && a.zout64 != nullptr) a.zout64[row] = static_cast<double>(w);
}

template <typename T, bool GEN, bool TWO>
__device__ __forceinline__ void update_first_body(const PassArgs<T> &a, double *x, const double *p, const double *q,
                                                  double *r) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ T s_w[kTileRows];
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  const int ns = a.g.ns;
  const StageLayout L = update_first_layout<T>(a.g);
  load_patterns(s_pat, a.pat, a.g.npat);
  ring_init(R, ns);
  if (threadIdx.x >= kConsumers) {
    const ChunkCtx ck{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      // x (v1) and q (v3) are not read again before the next x/r update
      produce<T, double, double, double, true, double, 0xAu>(R, st, a.td, tile, a.g, L, smem + st * L.bytes,
                                                             a.ib_sp, a.ib_col, a.ib_val, a.meta, r,
                                                             kUfDirect ? nullptr : x, p, kUfDirect ? nullptr : q,
                                                             part);
    };
    auto gated = [&]() { return gated_off(a); };
    if (TWO && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, 1, a.td);
    else if (threadIdx.x == kConsumers)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, 1, a.td);
    else
      pdl_wait();
    if (gated_off(a)) return;
  } else {
    pdl_wait();
    if (gated_off(a)) return;
    if (threadIdx.x == 0) tl_mark(a.st, 2, 0, false);
    const double alpha = a.st->alpha;
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * L.bytes;
      const bool ok = R.ok[st] != 0;
      if (!GEN && kRowsPerThread == 1 && kFastTiles && ok && ((d.hi - d.lo) & 31) == 0 && (d.lo & 31) == 0 &&
          a.g.kib <= 7) {
        const double *xs = kUfDirect ? x + d.lo : staged(sb + L.v1, x, d.lo, d.hi);
        const double *ps = staged(sb + L.v2, p, d.lo, d.hi);
        const double *qs = kUfDirect ? q + d.lo : staged(sb + L.v3, q, d.lo, d.hi);
        const double *rs = staged(sb + L.v0, r, d.lo, d.hi);
        const T *val = reinterpret_cast<const T *>(sb + L.val);
        const int *spp = staged(sb + L.sp, a.ib_sp, d.s0, d.s1 + 1);
        const uint16_t *mt = staged(sb + L.meta, a.meta, d.lo, d.hi);
        if (a.g.kib <= 3)
          update_first_full<T, 3>(a, tile, d, alpha, x, r, xs, ps, qs, rs, val, spp, mt, s_pat, s_w, ws);
        else
          update_first_full<T, 7>(a, tile, d, alpha, x, r, xs, ps, qs, rs, val, spp, mt, s_pat, s_w, ws);
        ring_release(R, st);
        continue;
      }
      double sq[kRowsPerThread];
      T rv[kRowsPerThread];
#pragma unroll
      for (int k = 0; k < kRowsPerThread; k++) {
        const int i = threadIdx.x + k * kConsumers, row = d.lo + i;
        sq[k] = 0.0;
        rv[k] = T(0);
        if (row >= d.hi) continue;
        const double xv = (ok && !kUfDirect) ? staged(sb + L.v1, x, d.lo, d.hi)[i] : x[row];
        const double pv = ok ? staged(sb + L.v2, p, d.lo, d.hi)[i] : p[row];
        const double qv = (ok && !kUfDirect) ? staged(sb + L.v3, q, d.lo, d.hi)[i] : q[row];
        const double ro = ok ? staged(sb + L.v0, r, d.lo, d.hi)[i] : r[row];
        st_evict_first(x + row, __dadd_rn(xv, __dmul_rn(alpha, pv)));  // (read again by the next update only)
        const double rn = __dsub_rn(ro, __dmul_rn(alpha, qv));
        r[row] = rn;
        sq[k] = __dmul_rn(rn, rn);
        rv[k] = narrow_checked(a, rn, row, true);
      }
      const double tot = tile_tree_rows(sq, ws, kBarConsumers);
      if (threadIdx.x == 0) put_part(a.part + tile, tot);
      const bool scols = ok && a.g.cols && d.ngen > 0;
      const int *col = scols ? reinterpret_cast<const int *>(sb + L.col) : a.ib_col + d.ie0;
      if (ok)
        bjac_first_body<T, GEN>(a, d, col, reinterpret_cast<const T *>(sb + L.val),
                           staged(sb + L.sp, a.ib_sp, d.s0, d.s1 + 1), staged(sb + L.meta, a.meta, d.lo, d.hi), rv,
                           s_pat, s_w);
      else
        bjac_first_body<T, GEN>(a, d, col, a.ib_val + d.ie0, a.ib_sp + d.s0, a.meta + d.lo, rv, s_pat, s_w);
      ring_release(R, st);
    }
    if (threadIdx.x == 0) tl_mark(a.st, 2, 1, true);
  }
  pdl_trigger();
  finish_grid<8, kFinRptWs>(a.st, 2, kStepRrZ, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);  // 16: a CTA per SM less
}

// One-level order: ptxas' own register budget (40, 5 CTAs per SM; an
// explicit minimum of 5 measured 1 % slower).  Two-level: the owners'
// polling code would raise the budget, so the one-level occupancy (5 CTAs
// per SM in fp32, 4 in fp64) is imposed.
template <typename T, bool GEN>
__global__ void __launch_bounds__(kWsThreads) k_update_first(const PassArgs<T> a, double *x, const double *p,
                                                             const double *q, double *r) {
  update_first_body<T, GEN, false>(a, x, p, q, r);
}
template <typename T, bool GEN>
__global__ void __launch_bounds__(kWsThreads, sizeof(T) == 4 ? 5 : 4)
    k_update_first_two(const PassArgs<T> a, double *x, const double *p, const double *q, double *r) {
  update_first_body<T, GEN, true>(a, x, p, q, r);
}

// Warp-per-tile fused x/r update + next first pass (same arithmetic and
// tile order as update_first_body; see k_bjac_wt for the warp-per-tile
// scheme).  Plans with generic rows keep k_update_first.
template <typename T, bool TWO>
__global__ void __launch_bounds__(kWtWarps * 32 + 32)
    k_update_first_wt(const PassArgs<T> a, double *x, const double *p, const double *q, double *r) {
  constexpr int NC = kWtWarps * 32;
  constexpr int kFinRpt = NC >= kFinThreads ? 1 : kFinThreads / NC;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ RingT<kWtMaxStages> R;
  __shared__ T s_w[kWtWarps][kTileRows];
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  const int ns = a.g.ns;
  const StageLayout L = update_first_layout<T>(a.g);
  load_patterns(s_pat, a.pat, a.g.npat);
  ring_init(R, ns, 32);
  if (threadIdx.x >= NC) {
    const ChunkCtx ck{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0};
    auto fill = [&](int st, int tile, int part) {
      // x (v1) and q (v3) are not read again before the next x/r update
      produce<T, double, double, double, true, double, 0xAu>(R, st, a.td, tile, a.g, L, smem + st * L.bytes,
                                                             a.ib_sp, a.ib_col, a.ib_val, a.meta, r,
                                                             kUfDirect ? nullptr : x, p, kUfDirect ? nullptr : q,
                                                             part);
    };
    auto gated = [&]() { return gated_off(a); };
    if (TWO && ck.poll)
      producer_loop(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, ck, kWtWarps, a.td);
    else if (threadIdx.x == NC)
      producer_loop_single(R, a.g.ntiles, ns, a.ctr, a.prefetch != 0, gated, fill, kWtWarps, a.td);
    else
      pdl_wait();
    if (gated_off(a)) return;
  } else {
    pdl_wait();
    if (gated_off(a)) return;
    const double alpha = a.st->alpha;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T *sw = s_w[c];
    int st = c, phase = 0;
    for (;;) {
      mbar_wait(&R.full[st], phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * L.bytes;
      const bool ok = R.ok[st] != 0;
      const double *xs = (ok && !kUfDirect) ? staged(sb + L.v1, x, d.lo, d.hi) : x + d.lo;
      const double *ps = ok ? staged(sb + L.v2, p, d.lo, d.hi) : p + d.lo;
      const double *qs = (ok && !kUfDirect) ? staged(sb + L.v3, q, d.lo, d.hi) : q + d.lo;
      const double *rs = ok ? staged(sb + L.v0, r, d.lo, d.hi) : r + d.lo;
      double sq[kWtRows];
      T rv[kWtRows];
#pragma unroll
      for (int k = 0; k < kWtRows; k++) {
        const int i = lane + 32 * k, row = d.lo + i;
        sq[k] = 0.0;
        rv[k] = T(0);
        if (row >= d.hi) continue;
        st_evict_first(x + row, __dadd_rn(xs[i], __dmul_rn(alpha, ps[i])));  // (read again by the next update only)
        const double rn = __dsub_rn(rs[i], __dmul_rn(alpha, qs[i]));
        r[row] = rn;
        sq[k] = __dmul_rn(rn, rn);
        rv[k] = narrow_checked(a, rn, row, true);
      }
      const double tot = wt_tile_sum(sq);
      if (lane == 0) put_part(a.part + tile, tot);
      const T *val = ok ? reinterpret_cast<const T *>(sb + L.val) : a.ib_val + d.ie0;
      const int *spp = ok ? staged(sb + L.sp, a.ib_sp, d.s0, d.s1 + 1) : a.ib_sp + d.s0;
      const uint16_t *mt = ok ? staged(sb + L.meta, a.meta, d.lo, d.hi) : a.meta + d.lo;
      wt_first_tile<T>(a, d, val, spp, mt, rv, s_pat, sw);
      if (lane == 0) mbar_arrive(&R.empty[st]);
      st += kWtWarps;
      if (st >= ns) {
        st -= ns;
        phase ^= 1;
      }
    }
  }
  pdl_trigger();
  finish_grid<8, kFinRpt>(a.st, 2, kStepRrZ, ChunkCtx{a.csum, a.part, a.g.ntiles, TWO ? a.g.poll : 0}, ws);
}

// ---------------------------------------------------------------------------
// Wave kernel (fixed-branch policies, k = 2): the x/r update + next first
// pass of iteration i and the last pass of iteration i+1 in ONE kernel.
// No global reduction sits between them: the last pass of tile m needs r of
// its own rows and z1 of the rows its pattern offsets reach (tiles within
// `reach` of m).  Work items are claimed in the order
//   U(0) .. U(lag-1), then U(lag) L(0) U(lag+1) L(1) ..., then the last L's
// (U = update + first pass of a tile, L = last pass), so with lag > reach
// every item an L item depends on was claimed before it; U items never wait,
// hence the walk cannot deadlock (only CTAs that claimed an item hold one).
// A U item is published when its producer recycles the stage (the consumers'
// mbarrier release, the producer's acquire, then a gpu-scope release
// increment of the item's tile-group counter); an L item's consumers wait
// (acquire) until every group it reaches is complete for this launch, then
// read r and z1 with coherent loads.  The r.r and r.z sums keep their tile
// order; the final CTA runs the relres step of iteration i and, unless the
// solve stopped there, the rho step of iteration i+1 -- the same steps the
// separate kernels ran, so the solve is bit-identical.
// ---------------------------------------------------------------------------
struct WaveCtl {
  unsigned int *gcnt;  // per tile group: U items published (cumulative over the solve)
  const int2 *dep;     // per tile: first and last tile group its last pass reads
  int lag;             // U items ahead of the L items
  int gshift;          // tile group = tile >> gshift
  int dbg;             // experiments (MPB_WAVE_DBG): 1 no dependency waits (unsafe), 2 relaxed publish
                       // (unsafe), 4 count the wait polls in gcnt[spin_slot]
  int spin_slot;
};

__device__ __forceinline__ int2 wave_item(int j, int nt, int lag) {  // (kind 0 U / 1 L, tile)
  if (j < lag) return make_int2(0, j);
  const int k = j - lag, nb = 2 * (nt - lag);
  if (k < nb) return (k & 1) ? make_int2(1, k >> 1) : make_int2(0, lag + (k >> 1));
  return make_int2(1, nt - lag + (k - nb));
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T, int KS, int KI>
__global__ void __launch_bounds__(kTileThreads + 32)
    k_wave(const PassArgs<T> au, const PassArgs<T> al, double *x, const double *p, const double *q, double *r,
           const WaveCtl wc) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Ring R;
  __shared__ int s_kind[kMaxStages];
  __shared__ T s_w[kTileRows];
  __shared__ double ws[32];
  __shared__ int s_pat[kPatMax * kPatStride];
  const int ns = au.g.ns, nt = au.g.ntiles;
  const StageLayout Lu = update_first_layout<T>(au.g);
  const StageLayout Ll = stage_layout(al.g.cap_e, sizeof(T), al.g.max_sl, false, true, 0, 0, 0);
  const uint32_t sbytes = max(Lu.bytes, Ll.bytes);
  load_patterns(s_pat, au.pat, au.g.npat);
  ring_init(R, ns);
  if (threadIdx.x >= kTileThreads) {  // producer warp (lane 0 walks the items)
    pdl_wait();
    if (gated_off(au)) return;
    if (threadIdx.x != kTileThreads) return;
    const unsigned int total = 2u * static_cast<unsigned int>(nt);
    auto claim = [&]() -> int {
      const unsigned int v = atomicAdd(au.ctr, 1u);
      if (v == total + gridDim.x - 1u) atomicExch(au.ctr, 0u);
      return v < total ? static_cast<int>(v) : -1;
    };
    auto publish_tile = [&](int tile) {  // a finished U item (its stage's empty barrier acquired)
      if (wc.dbg & 2)
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(wc.gcnt + (tile >> wc.gshift)) : "memory");
      else
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(wc.gcnt + (tile >> wc.gshift)) : "memory");
    };
    auto publish = [&](int s) {
      if (s_kind[s] == 0 && R.tile[s] >= 0) publish_tile(R.tile[s]);
    };
    auto fill = [&](int s, int2 it) {
      unsigned char *stage = smem + s * sbytes;
      R.tile[s] = it.y;
      s_kind[s] = it.x;
      if (it.x == 0)
        produce<T, double, double, double, true, double, 0xAu>(R, s, au.td, it.y, au.g, Lu, stage, au.ib_sp,
                                                               au.ib_col, au.ib_val, au.meta, r, x, p, q);
      else
        produce<T, double, double, double>(R, s, al.td, it.y, al.g, Ll, stage, al.sp, al.scol, al.sval, al.meta,
                                           static_cast<const double *>(nullptr), static_cast<const double *>(nullptr),
                                           static_cast<const double *>(nullptr));
    };
    int st = 0, rnd = 0;
    int cur = claim();
    for (;;) {
      int done_tile = -1;  // U item the consumers just finished in stage st
      if (rnd > 0) {
        mbar_wait_sleep(&R.empty[st], (rnd - 1) & 1);
        if (s_kind[st] == 0) done_tile = R.tile[st];
      }
      if (cur < 0) {
        if (done_tile >= 0) publish_tile(done_tile);
        break;
      }
      const int2 it = wave_item(cur, nt, wc.lag);
      fill(st, it);  // the refill's copies first, then the (fenced) publication
      if (done_tile >= 0) publish_tile(done_tile);
      cur = claim();
      if (cur >= 0) prefetch_desc(au.td, wave_item(cur, nt, wc.lag).y);
      if (++st == ns) {
        st = 0;
        rnd++;
      }
    }
    R.tile[st] = -1;  // end marker (stage st is free)
    mbar_arrive(&R.full[st]);
    // publish the items still in flight, in the consumers' order
    for (int k = 1; k < ns; k++) {
      const int s = (st + k) % ns;
      const int fills = s > st ? rnd : rnd + 1;  // times stage s was filled
      if (fills == 0) continue;
      mbar_wait_sleep(&R.empty[s], (fills - 1) & 1);
      publish(s);
    }
  } else {
    pdl_wait();
    if (gated_off(au)) return;
    const double alpha = au.st->alpha;
    const unsigned int epoch1 = static_cast<unsigned int>(au.st->wave_epoch) + 1u;
    for (RingCursor cur;; cur.advance(ns)) {
      const int st = cur.st;
      mbar_wait(&R.full[st], cur.phase);
      const int tile = R.tile[st];
      if (tile < 0) break;
      const TileDesc d = R.desc[st];
      const unsigned char *sb = smem + st * sbytes;
      if (s_kind[st] == 0) {
        update_first_full<T, KI>(au, tile, d, alpha, x, r, staged(sb + Lu.v1, x, d.lo, d.hi),
                                 staged(sb + Lu.v2, p, d.lo, d.hi), staged(sb + Lu.v3, q, d.lo, d.hi),
                                 staged(sb + Lu.v0, r, d.lo, d.hi), reinterpret_cast<const T *>(sb + Lu.val),
                                 staged(sb + Lu.sp, au.ib_sp, d.s0, d.s1 + 1), staged(sb + Lu.meta, au.meta, d.lo, d.hi),
                                 s_pat, s_w, ws);
      } else {
        if (threadIdx.x < 32 && !(wc.dbg & 1)) {  // every tile group the pass reads: complete for this launch
          const int2 dg = wc.dep[tile];
          for (int g = dg.x + static_cast<int>(threadIdx.x); g <= dg.y; g += 32) {
            const unsigned int gsz = static_cast<unsigned int>(min(1 << wc.gshift, nt - (g << wc.gshift)));
            const unsigned int target = epoch1 * gsz;
            while (ld_acquire_u32(wc.gcnt + g) < target) {
              if (wc.dbg & 4) atomicAdd(wc.gcnt + wc.spin_slot, 1u);
              __nanosleep(64);
            }
          }
        }
        named_sync(kBarConsumers, kTileThreads);
        bjac_tile_full<T, true, KS, KI, false, true>(al, tile, d, reinterpret_cast<const T *>(sb + Ll.val),
                                                    staged(sb + Ll.sp, al.sp, d.s0, d.s1 + 1),
                                                    staged(sb + Ll.meta, al.meta, d.lo, d.hi), al.r64 + d.lo,
                                                    s_pat, s_w, ws);
      }
      ring_release(R, st);
    }
  }
  pdl_trigger();
  // final CTA: relres step of iteration i, then (unless the solve stopped) rho of i+1
  SolverState *gst = au.st;
  if (!grid_last(&gst->ticket[2])) return;
  __shared__ __align__(16) unsigned long long s_state[kStWords];
  if (threadIdx.x < kStWords) s_state[threadIdx.x] = __ldcg(reinterpret_cast<const unsigned long long *>(gst) + threadIdx.x);
  SolverState *L = reinterpret_cast<SolverState *>(s_state);
  const double rr = fin_sum<8, 1>(au.part, nt, ws);  // (its barriers publish s_state)
  if (threadIdx.x == 0) scalar_step_body(kStepRrZ, rr, L);
  __syncthreads();
  if (!L->done) {
    const double rz = fin_sum<8, 1>(al.part, nt, ws);
    if (threadIdx.x == 0) scalar_step_body(kStepRho, rz, L);
  }
  if (threadIdx.x == 0) {
    L->wave_epoch++;
    gst->ticket[2] = 0u;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // the changed state back (state_store's ranges)
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(gst);
    constexpr int a1 = static_cast<int>(offsetof(SolverState, tr_relres) / 8);
    constexpr int b0 = static_cast<int>(offsetof(SolverState, dist) / 8), b1 = static_cast<int>(offsetof(SolverState, cond) / 8);
    for (int i = threadIdx.x; i < a1 + (b1 - b0); i += 32) {
      const int w = i < a1 ? i : b0 + (i - a1);
      dst[w] = s_state[w];
    }
  }
}

// res = b - A x (or b), optionally stored; res.res partial; the last CTA runs
// `step` (R0 / True / Final) when st != null.
// gate: 0 always, 1 only when st->true_pending (strided true residual)
template <bool HAS_X>
__global__ void __launch_bounds__(kCtaThreads)
    k_resid(const int *sp, const int *scol, const double *sval, const TileDesc *td, int ntiles, const double *b,
            const double *x, double *rout, double *part, SolverState *st, int gate, int step, double *csum,
            int poll) {
  if (gate == 1 && (st == nullptr || !st->true_pending)) return;
  __shared__ double ws[32];
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const TileDesc d = td[tile];
    const int row = d.lo + threadIdx.x;
    double sq = 0.0;
    if (row < d.hi) {
      double res = b[row];
      if (HAS_X) {
        const int s = row >> 5, sb = sp[s], width = (sp[s + 1] - sb) >> 5, base = sb + (row & 31);
        double ax = 0.0;
        for (int j0 = 0; j0 < width; j0 += kSlots) {
          int c[kSlots];
          double v[kSlots], g[kSlots];
#pragma unroll
          for (int u = 0; u < kSlots; u++) {
            const bool ok = j0 + u < width;
            c[u] = ok ? __ldg(scol + base + 32 * (j0 + u)) : -1;
            v[u] = ok ? __ldg(sval + base + 32 * (j0 + u)) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kSlots; u++) g[u] = c[u] >= 0 ? __ldg(x + c[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < kSlots; u++)
            if (c[u] >= 0) ax = __dadd_rn(ax, __dmul_rn(v[u], g[u]));
        }
        res = __dsub_rn(res, ax);
      }
      if (rout != nullptr) rout[row] = res;
      sq = __dmul_rn(res, res);
    }
    const double tot = block_tree<kTileThreads>(sq, ws);
    if (threadIdx.x == 0) put_part(part + tile, tot);
  }
  const ChunkCtx ck{st != nullptr ? csum : nullptr, part, ntiles, poll};
  chunk_duties_strided(ck, blockIdx.x, gridDim.x);
  finish_grid(st, 3, step, ck, ws);
}

// one-thread scalar step (solve start: wall-clock origin of the trace)
__global__ void k_scalar_start(SolverState *st) {
  if (threadIdx.x == 0) {
    SolverState L;
    state_load(L, st);
    scalar_step(kStepStart, 0.0, &L);
    state_store(st, L);
  }
}

__global__ void k_fill(double *p, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------------------------
// SELL-32 construction: slice s of rows [32s, 32s+32), entry j of row r at
// sp[s] + 32 j + r % 32 (padding: column -1 / value 0, set by memset)
// ---------------------------------------------------------------------------
template <typename E>
__global__ void k_sell_pack(long long n, const int *rp, const int *sp, const E *csr, E *sell) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int base = sp[r >> 5] + static_cast<int>(r & 31);
    const int s = rp[r], len = rp[r + 1] - s;
    for (int j = 0; j < len; j++) sell[base + 32 * j] = csr[s + j];
  }
}

// ---- row patterns (setup, per SELL structure) --------------------------------
// The row's stored columns as offsets from the row, in stored order, and a
// 64-bit key of (length, offsets); key 0 = no pattern (longer than kSlots).
__device__ __forceinline__ unsigned long long row_pattern(const int *sp, const int *scol, int row, int (&off)[kSlots],
                                                          int &len) {
  const int s = row >> 5, sb = sp[s], width = (sp[s + 1] - sb) >> 5, base = sb + (row & 31);
  len = 0;
  for (int j = 0; j < width; j++) {
    const int c = scol[base + 32 * j];
    if (c < 0) break;
    if (j < kSlots) off[j] = c - row;
    len = j + 1;
  }
  if (len > kSlots) return 0ull;
  unsigned long long h = 0x9E3779B97F4A7C15ull ^ static_cast<unsigned long long>(len);
  for (int j = 0; j < len; j++) {
    h ^= static_cast<unsigned int>(off[j]);
    h *= 0x100000001B3ull;
    h ^= h >> 29;
  }
  return h | 1ull;
}

// count the rows of every pattern into an open-addressing table (one atomic
// per distinct pattern per warp)
__global__ void k_pat_insert(long long n, const int *sp, const int *scol, PatSlot *tab) {
  const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  int off[kSlots], len = 0;
  const unsigned long long key = r < n ? row_pattern(sp, scol, static_cast<int>(r), off, len) : 0ull;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  if (key == 0ull || (threadIdx.x & 31) != __ffs(peers) - 1) return;
  unsigned s = static_cast<unsigned>(key) & (kPatHash - 1);
  for (int probe = 0; probe < kPatHash; probe++, s = (s + 1) & (kPatHash - 1)) {
    unsigned long long k = *reinterpret_cast<volatile unsigned long long *>(&tab[s].key);
    if (k == 0ull) {
      k = atomicCAS(&tab[s].key, 0ull, key);
      if (k == 0ull) {
        tab[s].rep = static_cast<int>(r);
        k = key;
      }
    }
    if (k == key) {
      atomicAdd(&tab[s].count, __popc(peers));
      return;
    }
  }
}

// table entries of the chosen patterns from one representative row each
__global__ void k_pat_fetch(const int *reps, int npat, const int *sp, const int *scol, int *pat) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npat) return;
  const int row = reps[i];
  int off[kSlots], len = 0;
  row_pattern(sp, scol, row, off, len);
  int dpos = 255;
  for (int j = 0; j < len; j++)
    if (off[j] == 0) dpos = j;
  pat[i * kPatStride] = len | (dpos << 8);
  for (int j = 0; j < kSlots; j++) pat[i * kPatStride + 1 + j] = j < len ? off[j] : 0;
}

// each row's pattern id (verified entry by entry) or kPidGeneric
__global__ void k_pat_assign(long long n, const int *sp, const int *scol, const PatSlot *tab, const int *slot_pid,
                             const int *pat, uint8_t *pid) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    int off[kSlots], len = 0;
    const unsigned long long key = row_pattern(sp, scol, static_cast<int>(r), off, len);
    uint8_t out = kPidGeneric;
    if (key != 0ull) {
      unsigned s = static_cast<unsigned>(key) & (kPatHash - 1);
      int cand = -1;
      for (int probe = 0; probe < kPatHash; probe++, s = (s + 1) & (kPatHash - 1)) {
        const unsigned long long k = tab[s].key;
        if (k == key) {
          cand = slot_pid[s];
          break;
        }
        if (k == 0ull) break;
      }
      if (cand >= 0) {
        const int *P = pat + cand * kPatStride;
        bool same = pat_len(P[0]) == len;
        for (int j = 0; j < len; j++) same = same && P[1 + j] == off[j];
        if (same) out = static_cast<uint8_t>(cand);
      }
    }
    pid[r] = out;
  }
}

// Per-row static structure against a block partition (plan-bound): pattern
// id and in-block slot range, or kMetaGeneric (no pattern, no stored
// diagonal, or in-block entries not one contiguous slot range).
__global__ void k_build_meta(long long n, const uint8_t *pid, const int *pat, const int *boff, int nb,
                             uint16_t *meta) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(r);
    uint16_t m = kMetaGeneric;
    const int id = pid[row];
    if (id != kPidGeneric) {
      const int *P = pat + id * kPatStride;
      const int len = pat_len(P[0]), dpos = pat_dpos(P[0]);
      int L = 0, H = nb;
      while (H - L > 1) {
        const int M = (L + H) >> 1;
        if (boff[M] <= row) L = M; else H = M;
      }
      const int blo = boff[L], bhi = boff[L + 1];
      // in-block entries form one contiguous slot range (columns ascend in
      // global order; multi-GPU ghost renumbering keeps the stored order and
      // maps only out-of-slab columns, which are never in-block)
      int i0 = -1, i1 = -1, nin = 0;
      for (int j = 0; j < len; j++) {
        const int c = row + P[1 + j];
        if (c >= blo && c < bhi) {
          if (i0 < 0) i0 = j;
          i1 = j + 1;
          nin++;
        }
      }
      if (i0 < 0) i0 = i1 = 0;
      if (dpos < len && nin == i1 - i0 && i1 <= 15)
        m = static_cast<uint16_t>(id | (i0 << 8) | (i1 << 12));
    }
    meta[row] = m;
  }
}

// generic rows per tile (TileDesc::ngen)
__global__ void k_tile_generic(TileDesc *td, const uint16_t *meta) {
  const TileDesc d = td[blockIdx.x];
  const int row = d.lo + threadIdx.x;
  const int gen = __syncthreads_count(row < d.hi && meta[row] == kMetaGeneric);
  if (threadIdx.x == 0) td[blockIdx.x].ngen = gen;
}

// In-block entries of each row (columns inside the row's block): count, and
// packing into the plan's in-block SELL-32 layout (same slices, widths =
// longest in-block row of the slice), in ascending column order.
__device__ __forceinline__ void row_block(const int *boff, int nb, int row, int &blo, int &bhi) {
  int L = 0, H = nb;
  while (H - L > 1) {
    const int M = (L + H) >> 1;
    if (boff[M] <= row) L = M; else H = M;
  }
  blo = boff[L];
  bhi = boff[L + 1];
}

__global__ void k_ib_count(long long n, const int *sp, const int *scol, const int *boff, int nb, int *cnt) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(r);
    const int s = row >> 5, sb = sp[s], width = (sp[s + 1] - sb) >> 5, base = sb + (row & 31);
    int blo, bhi;
    row_block(boff, nb, row, blo, bhi);
    int k = 0;
    for (int j = 0; j < width; j++) {
      const int c = scol[base + 32 * j];
      k += (c >= blo && c < bhi) ? 1 : 0;
    }
    cnt[row] = k;
  }
}

template <typename E>
__global__ void k_ib_pack(long long n, const int *sp, const int *scol, const int *boff, int nb, const int *ib_sp,
                          const E *src, E *dst) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int row = static_cast<int>(r);
    const int s = row >> 5, sb = sp[s], width = (sp[s + 1] - sb) >> 5, base = sb + (row & 31);
    const int ibase = ib_sp[s] + (row & 31);
    int blo, bhi;
    row_block(boff, nb, row, blo, bhi);
    int k = 0;
    for (int j = 0; j < width; j++) {
      const int c = scol[base + 32 * j];
      if (c >= blo && c < bhi) dst[ibase + 32 * (k++)] = src[base + 32 * j];
    }
  }
}

// ---------------------------------------------------------------------------
// GPU-side problem assembly (problems.py restated): the
// 7-point finite-volume operator from a cell field kappa, and the SplitMix64
// uniform stream.  Same IEEE operations in the same order as the host
// generators (no FMA), so the matrices and vectors are bit-identical.
// ---------------------------------------------------------------------------
// entries of rows [0, p) of the n^3 7-point operator: 7 p minus the missing
// neighbours of those rows (closed form: no scan)
__host__ __device__ inline long long stencil_row_ptr(long long p, long long n) {
  const long long n2 = n * n, L = p / n, P = p / n2, rem = p % n2;
  const long long mx = 2 * L + (p % n > 0 ? 1 : 0);
  const long long my = 2 * n * P + (rem < n ? rem : n) + (rem > n * (n - 1) ? rem - n * (n - 1) : 0);
  const long long mz = (p < n2 ? p : n2) + (p > (n - 1) * n2 ? p - (n - 1) * n2 : 0);
  return 7 * p - mx - my - mz;
}

__device__ __forceinline__ double harmonic_face(double w, double a, double b) {
  return __dmul_rn(w, __ddiv_rn(__dmul_rn(__dmul_rn(2.0, a), b), __dadd_rn(a, b)));  // problems.py _harmonic
}

// Row p: entries zm, ym, xm, diag, xp, yp, zp (ascending column), the
// off-diagonals -(face*scale), the diagonal ((((xm+xp)+ym)+yp)+zm)+zp)*scale.
// Config 4 (3-temperature system, problems.py three_temperature): cell p's
// 7-point row (rp1/col1/val1 of the D field) becomes rows 3p+c, c = 0..2:
// [lower stencil entries] [cell block] [upper stencil entries], the cell
// block  c=0: diag, (3p+1, -w_re);  c=1: (3p, -w_re), diag, (3p+2, -w_ei);
// c=2: (3p+1, -w_ei), diag; diagonal = ((stencil diag + tt) [+ w_re]) [+ w_ei]
// in that order.  Row offsets are closed-form: cell p's rows start at
// 3 rp1[p] + 4 p (4 coupling entries per cell).
__global__ void k_expand_3t(long long ncell, const int *rp1, const int *col1, const double *val1, const double *wre,
                            const double *wei, double tt, int *rp3, int *col3, double *val3) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < ncell;
       p += (long long)gridDim.x * blockDim.x) {
    const int b1 = rp1[p], cnt = rp1[p + 1] - b1;
    int nlo = 0;
    while (col1[b1 + nlo] != static_cast<int>(p)) nlo++;
    const long long R = 3LL * b1 + 4LL * p;
    const double wr = wre[p], we = wei[p];
    for (int c = 0; c < 3; c++) {
      const long long start = R + static_cast<long long>(c) * cnt + (c == 0 ? 0 : (c == 1 ? 1 : 3));
      const int cpl = c == 1 ? 2 : 1;
      rp3[3 * p + c] = static_cast<int>(start);
      for (int j = 0; j < cnt; j++) {
        if (j == nlo) continue;
        const long long dst = start + j + (j > nlo ? cpl : 0);
        col3[dst] = 3 * col1[b1 + j] + c;
        val3[dst] = val1[b1 + j];
      }
      const long long blk = start + nlo;
      double dd = __dadd_rn(val1[b1 + nlo], tt);
      if (c <= 1) dd = __dadd_rn(dd, wr);
      if (c >= 1) dd = __dadd_rn(dd, we);
      const int cell3 = static_cast<int>(3 * p);
      if (c == 0) {
        col3[blk] = cell3;
        val3[blk] = dd;
        col3[blk + 1] = cell3 + 1;
        val3[blk + 1] = -wr;
      } else if (c == 1) {
        col3[blk] = cell3;
        val3[blk] = -wr;
        col3[blk + 1] = cell3 + 1;
        val3[blk + 1] = dd;
        col3[blk + 2] = cell3 + 2;
        val3[blk + 2] = -we;
      } else {
        col3[blk] = cell3 + 1;
        val3[blk] = -we;
        col3[blk + 1] = cell3 + 2;
        val3[blk + 1] = dd;
      }
    }
    if (p == ncell - 1) rp3[3 * ncell] = static_cast<int>(3LL * rp1[ncell] + 4LL * ncell);
  }
}

__global__ void k_stencil(long long n, const double *kap, double wx, double wy, double wz, double scale, int *rp,
                          int *col, double *val) {
  const long long N = n * n * n, n2 = n * n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const long long i = p % n, j = (p / n) % n, k = p / n2;
    const double kc = kap[p];
    const double fxm = i > 0 ? harmonic_face(wx, kap[p - 1], kc) : __dmul_rn(wx, kc);
    const double fxp = i < n - 1 ? harmonic_face(wx, kc, kap[p + 1]) : __dmul_rn(wx, kc);
    const double fym = j > 0 ? harmonic_face(wy, kap[p - n], kc) : __dmul_rn(wy, kc);
    const double fyp = j < n - 1 ? harmonic_face(wy, kc, kap[p + n]) : __dmul_rn(wy, kc);
    const double fzm = k > 0 ? harmonic_face(wz, kap[p - n2], kc) : __dmul_rn(wz, kc);
    const double fzp = k < n - 1 ? harmonic_face(wz, kc, kap[p + n2]) : __dmul_rn(wz, kc);
    long long e = stencil_row_ptr(p, n);
    rp[p] = static_cast<int>(e);
    if (p == N - 1) rp[N] = static_cast<int>(stencil_row_ptr(N, n));
    const double d = __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(fxm, fxp), fym), fyp), fzm), fzp),
                               scale);
    if (k > 0) { col[e] = static_cast<int>(p - n2); val[e++] = -__dmul_rn(fzm, scale); }
    if (j > 0) { col[e] = static_cast<int>(p - n); val[e++] = -__dmul_rn(fym, scale); }
    if (i > 0) { col[e] = static_cast<int>(p - 1); val[e++] = -__dmul_rn(fxm, scale); }
    col[e] = static_cast<int>(p);
    val[e++] = d;
    if (i < n - 1) { col[e] = static_cast<int>(p + 1); val[e++] = -__dmul_rn(fxp, scale); }
    if (j < n - 1) { col[e] = static_cast<int>(p + n); val[e++] = -__dmul_rn(fyp, scale); }
    if (k < n - 1) { col[e] = static_cast<int>(p + n2); val[e] = -__dmul_rn(fzp, scale); }
  }
}

// problems.py splitmix64_stream: state_i = seed + (i+1) gamma, mixed, top 53 bits / 2^53
__global__ void k_splitmix64(unsigned long long seed, long long count, double a, double b, double *out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + static_cast<unsigned long long>(i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    out[i] = a == 1.0 && b == 0.0 ? u : __dadd_rn(__dmul_rn(a, u), b);  // a*u + b (e.g. C1: 2u - 1)
  }
}

// ---------------------------------------------------------------------------
// reference backend kernels (plugin level; CSR; kernels_numba.py)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_matvec(long long n, const int *rp, const int *ci, const T *val, const T *x, T *y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++) acc = add_rn(acc, mul_rn(__ldg(val + e), __ldg(x + __ldg(ci + e))));
    y[i] = acc;
  }
}

template <typename T>
__global__ void k_msweep_init(long long rs, long long re, const T *r, const T *diag, T *y) {
  for (long long i = rs + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < re; i += (long long)gridDim.x * blockDim.x)
    y[i] = div_rn(r[i], diag[i]);
}
template <typename T>
__global__ void k_msweep_tmp(long long rs, long long re, const int *rp, const int *ci, const T *val,
                             const uint8_t *mask, const T *y, T *tmp) {
  for (long long i = rs + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < re; i += (long long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (mask[e]) acc = add_rn(acc, mul_rn(val[e], y[ci[e]]));
    tmp[i] = acc;
  }
}
template <typename T>
__global__ void k_msweep_upd(long long rs, long long re, const T *r, const T *diag, const T *tmp, T *y) {
  for (long long i = rs + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < re; i += (long long)gridDim.x * blockDim.x)
    y[i] = add_rn(y[i], div_rn(sub_rn(r[i], tmp[i]), diag[i]));
}

// inner_apply on one block [lo, hi): block-local vectors, mask = [lo, hi)
template <typename T>
__global__ void k_inner_init(int lo, int hi, const int *rp, const int *ci, const T *val, const T *rb, T *db, T *yb) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    T dd = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (ci[e] == i) dd = val[e];
    db[i - lo] = dd;
    yb[i - lo] = div_rn(rb[i - lo], dd);
  }
}
template <typename T>
__global__ void k_inner_sweep(int lo, int hi, const int *rp, const int *ci, const T *val, const T *rb, const T *db,
                              const T *ysrc, T *ydst) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++) {
      const int c = ci[e];
      if (c >= lo && c < hi) acc = add_rn(acc, mul_rn(val[e], ysrc[c - lo]));
    }
    ydst[i - lo] = add_rn(ysrc[i - lo], div_rn(sub_rn(rb[i - lo], acc), db[i - lo]));
  }
}

// per-tile sum of x*y (SQ: y ignored, x widened and squared); tile_lo may be
// null (uniform kTileRows-row tiles)
template <typename T, typename ACC, bool SQ>
__global__ void __launch_bounds__(kTileThreads)
    k_tile_dot(long long n, const int *tile_lo, const T *x, const T *y, ACC *part) {
  __shared__ ACC ws[32];
  long long lo, hi;
  if (tile_lo != nullptr) {
    lo = tile_lo[blockIdx.x];
    hi = tile_lo[blockIdx.x + 1];
  } else {
    lo = (long long)blockIdx.x * kTileRows;
    hi = lo + kTileRows < n ? lo + kTileRows : n;
  }
  ACC acc = ACC(0);
  for (long long i = lo + threadIdx.x; i < hi; i += kTileThreads) {
    if (SQ) {
      const ACC v = static_cast<ACC>(x[i]);
      acc = add_rn(acc, mul_rn(v, v));
    } else {
      acc = add_rn(acc, mul_rn(static_cast<ACC>(x[i]), static_cast<ACC>(y[i])));
    }
  }
  const ACC tot = block_tree<kTileThreads>(acc, ws);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// chunk sums of the two-level order (include/mpbjac_order.h): one warp per chunk
template <typename ACC>
__global__ void __launch_bounds__(kTileThreads) k_chunk_sums(const ACC *part, long long nparts, ACC *csum) {
  const long long c = (long long)blockIdx.x * (kTileThreads / 32) + (threadIdx.x >> 5);
  const long long nch = (nparts + kChunkTiles - 1) / kChunkTiles;
  if (c >= nch) return;
  const ACC v = chunk_sum_warp(part, c, nparts);
  if ((threadIdx.x & 31) == 0) csum[c] = v;
}

// the final level over `nparts` values (chunk sums)
template <typename ACC>
__global__ void __launch_bounds__(kFinThreads) k_fin(const ACC *part, long long nparts, ACC *out) {
  __shared__ ACC ws[32];
  ACC acc = ACC(0);
  for (long long i = threadIdx.x; i < nparts; i += kFinThreads) acc = add_rn(acc, part[i]);
  const ACC tot = block_tree<kFinThreads>(acc, ws);
  if (threadIdx.x == 0) *out = tot;
}

// RN-even narrowing with overflow count / first index (sparse.py:202-214)
__global__ void k_narrow(long long n, const double *src, float *dst, unsigned long long *cnt, long long *first) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = src[i];
    const float f = __double2float_rn(v);
    dst[i] = f;
    if (isinf(f) && isfinite(v)) {
      atomicAdd(cnt, 1ull);
      atomicMin(first, i);
    }
  }
}
__global__ void k_widen(long long n, const float *src, double *dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = static_cast<double>(src[i]);
}

// stored diagonal per row (bjac.py:171-185); missing / zero reported by row
template <typename T>
__global__ void k_setup_diag(long long n, const int *rp, const int *ci, const T *val, T *diag, long long *missing,
                             long long *zero) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    bool have = false;
    T dd = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (ci[e] == i) {
        have = true;
        dd = val[e];
      }
    diag[i] = dd;
    if (!have) atomicMin(missing, i);
    else if (dd == T(0)) atomicMin(zero, i);
  }
}

}  // namespace mpb
