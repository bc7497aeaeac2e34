// mpbjac.cu — C-ABI of libmpbjac.so (declared in include/mpbjac.h).
//
// Host side of the B200 hot path: tile plans, SELL-32 layouts, launch
// sequences for the fused preconditioner passes, and the device-resident
// PCG loop replayed as a CUDA graph.  Each entry point cites the reference
// function it replaces in include/mpbjac.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/mpbjac.h"
#include "mpbjac_kernels.cuh"
#include "mpbjac_features.cuh"

#include <cub/device/device_radix_sort.cuh>
#include "mpbjac_nccl.h"

using namespace mpb;

namespace {

constexpr int kDefaultGraphIters = 16;  // iterations per while-loop body (measured best: 16-32)
constexpr int kEltThreads = 256;

inline int status_of(cudaError_t e) { return e == cudaSuccess ? MPB_OK : static_cast<int>(e); }
// MPB_DEBUG_SYNC=1: synchronise the device after every launch and name it
inline void debug_sync(int line) {
  static const bool on = std::getenv("MPB_DEBUG_SYNC") != nullptr;
  if (!on) return;
  std::fprintf(stderr, "[mpb sync] launch at mpbjac.cu:%d ...", line);
  const cudaError_t e = cudaDeviceSynchronize();
  std::fprintf(stderr, " done (%d)\n", static_cast<int>(e));
}

#define MPB_CUDA(expr)                           \
  do {                                           \
    cudaError_t e_ = (expr);                     \
    if (e_ != cudaSuccess) return status_of(e_); \
  } while (0)

#define MPB_LAUNCHED(h)                          \
  do {                                           \
    (h)->launches++;                             \
    cudaError_t e_ = cudaGetLastError();         \
    if (e_ != cudaSuccess) return status_of(e_); \
    debug_sync(__LINE__);                        \
  } while (0)

struct GraphKey {
  const void *plan, *rp, *sell, *v64, *v32, *vop, *b, *x, *trr, *trt, *trb, *trw, *ws, *comm;
  int kind, k, t, iters, loop;
  long long stride, n;
  bool operator==(const GraphKey &o) const { return std::memcmp(this, &o, sizeof(GraphKey)) == 0; }
};

}  // namespace

struct mpb_plan {
  int device;
  int64_t n, nb, ntiles, max_tile_nnz;
  int large;
  int *d_tile_lo, *d_tile_bf, *d_tile_bl, *d_boff;
  TileDesc *d_td;         // per-tile descriptors (rows, SELL slices/entries, blocks)
  int max_tile_sell;      // max SELL entries of a tile
  int max_sl, max_nbk;    // max slices / blocks per tile
  int ub = 0;             // every block has this many rows (0: blocks differ)
  uint16_t *d_meta;       // per-row static structure (mpb_plan_bind_sell)
  const mpb_sell *bound;  // the SELL layout d_meta was built against
  int *d_ib_sp, *d_ib_col;  // in-block SELL layout (first passes)
  int64_t ib_nnz;
  int max_tile_ib;
  int max_ib_row;           // most in-block entries of a row (the sweeps' unroll bound)
  const int *d_pat;         // the bound SELL's row-pattern table (not owned)
  int npat;
  int ks;                   // compile-time slot count of the hot kernels (7 or 9)
  int64_t ngeneric;         // rows without a usable pattern (kMetaGeneric)
  WinSet win;               // z_in gather windows of the passes after the first (n == 0: none)
  // symmetric offset-slot SpMV (k_spmv_sym): the pattern offsets' nonnegative
  // half d[0..S) (S = 0: not eligible), per-pattern presence masks, and the
  // U layout built for one operator value array (sym_key)
  int sym_S = 0;
  int sym_d[8] = {};
  uint16_t *d_pmask = nullptr;
  double *d_U = nullptr;
  const void *sym_key = nullptr;
  bool sym_ok = false;
  // offset-slot ("DIA") layout of 7-point stencil plans with 64-row blocks
  // (k_bjac_dia): eligibility, the slot offsets, the slots that are in-block
  // somewhere, per-row masks, per-pattern slot maps, and where the DIA
  // values sit in the plan-packed value buffer (mpb_plan_pack_inblock_*)
  bool dia_layout = false;  // the arrays below exist (tile plans: dia_ok; large blocks: dia_big)
  bool dia_ok = false;      // tile kernels (blocks of 64 rows)
  bool dia_big = false;     // large-block kernels (k_big_dia_*)
  int dia_off[8] = {};
  int dia_ibany = 0;
  uint16_t *d_dmeta = nullptr;
  signed char *d_pslot = nullptr;
  int64_t dia_at = 0, dia_entries = 0;
  int64_t near_at = 0, near_entries = 0;  // the near slots alone (0 entries: some in-block entry sits elsewhere)
  // wave kernel (k_wave): eligibility, item lag, tile-group size and each
  // tile's dependency range in groups (mpb_plan_bind_sell)
  bool wave_ok = false;
  int wave_lag = 0, wave_gshift = 5, wave_ngroups = 0;
  int2 *d_wdep = nullptr;
};

// In-process group of slab ranks on one GPU (mpb_local_group_create): the
// ranks' host threads enqueue onto ONE shared stream, and every
// communication point (halo exchange, scalar-step all-reduce) is a host
// barrier at which rank 0 enqueues the whole exchange -- plain copies
// between the ranks' buffers, a rank-ordered sum kernel -- for all ranks.
// Nothing on the device waits on another rank: the stream serialises every
// rank's kernels.  It runs the multi-GPU code path (slabs, ghosts, halos,
// all-reduced scalar steps) with more ranks than GPUs, for tests.
struct LocalGroup {
  int nranks;
  cudaStream_t stream;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  // per-rank arguments of the current communication point
  struct Slot {
    void *buf;
    int es;
    int64_t n;
    mpb_halo halo;
    mpb::SolverState *st;
  };
  std::vector<Slot> slot;
  bool failed = false;  // a rank returned an error: the others leave their barriers
  // false: the group failed (the caller returns MPB_ERR_COMM)
  bool barrier(int rank = -1, const char *what = "") {
    static const bool dbg = std::getenv("MPB_DEBUG_LOCAL") != nullptr;
    if (dbg) std::fprintf(stderr, "[mpb local] rank %d barrier %s gen %lld\n", rank, what, generation);
    std::unique_lock<std::mutex> lk(mu);
    if (failed) return false;
    const long long gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      generation++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || failed; });
    }
    return !failed;
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    cv.notify_all();
  }
};

struct mpb_comm {
  mpb::ncclComm_t comm;
  int rank, nranks;
  LocalGroup *grp = nullptr;  // in-process group (no NCCL)
};

struct mpb_sell {
  int64_t n, nslices, nnz;  // nnz: padded entry count
  int *d_sp;                // nslices+1
  int *d_col;               // nnz
  uint8_t *d_pid;           // per-row pattern id or kPidGeneric
  int *d_pat;               // npat table entries of kPatStride ints
  int npat;
  int max_len;              // longest row pattern (slots)
};

struct mpb_handle {
  int device;
  cudaStream_t user;    // caller's stream (may be the legacy default stream)
  cudaStream_t solve;   // private stream for graph capture
  cudaEvent_t ev_in, ev_out, ev_t0, ev_t1;
  void *scratch;
  size_t scratch_bytes;
  SolverState *h_state;  // pinned
  unsigned int *d_ctr;   // tile-claim counters of the persistent kernels (reset by each launch)
  unsigned long long *d_tl;  // MPB_TIMELINE diagnostics buffer
  int64_t launches;
  cudaGraphExec_t gexec;
  cudaGraphConditionalHandle cond;  // while node of gexec (device-side solve loop)
  GraphKey gkey;
  int64_t graph_kernels;
  bool have_graph;
};

namespace {

int elt_blocks(long long n) {
  long long b = (n + kEltThreads - 1) / kEltThreads;
  return static_cast<int>(std::max(1LL, std::min(b, 148LL * 16)));
}

int ensure_scratch(mpb_handle *h, size_t bytes) {
  if (h->scratch_bytes >= bytes) return MPB_OK;
  if (h->scratch) {
    MPB_CUDA(cudaStreamSynchronize(h->user));
    MPB_CUDA(cudaFree(h->scratch));
    h->scratch = nullptr;
    h->scratch_bytes = 0;
  }
  bytes = std::max(bytes, size_t(1) << 20);
  MPB_CUDA(cudaMalloc(&h->scratch, bytes));
  h->scratch_bytes = bytes;
  return MPB_OK;
}

inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

// SELL-32 slice pointers from a host row_ptr (slice width = longest row of
// the slice); shared by mpb_sell_create and the plan's tile descriptors so
// both agree entry for entry.  Returns false if the layout exceeds int32.
bool sell_slice_ptrs(int64_t n, const int64_t *h_rp, std::vector<int> &sp) {
  const int64_t ns = (n + 31) / 32;
  sp.assign(ns + 1, 0);
  int64_t acc = 0;
  for (int64_t s = 0; s < ns; s++) {
    int64_t width = 0;
    const int64_t r1 = std::min<int64_t>(n, 32 * s + 32);
    for (int64_t r = 32 * s; r < r1; r++) width = std::max<int64_t>(width, h_rp[r + 1] - h_rp[r]);
    sp[s] = static_cast<int>(acc);
    acc += 32 * width;
    if (acc >= (int64_t(1) << 31)) return false;
  }
  sp[ns] = static_cast<int>(acc);
  return true;
}

constexpr int kStageCap = 4096;  // staged SELL entries per tile (2 stages per CTA)

// the two-level sum order applies (and chunk owners poll) above
// MPB_ONE_LEVEL_TILES tiles
bool owners_poll(int64_t ntiles) { return two_level(ntiles); }
// streamed one-level sums of the offset-slot kernels (defined with the workspace layout)
bool red_mode(const mpb_plan *p);
double *red_part(const mpb_plan *p, int64_t n, double *part);

template <typename T>
TileGeom geom_for(const mpb_plan *p) {
  TileGeom g;
  g.ntiles = static_cast<int>(p->ntiles);
  g.cap_e = std::min(p->max_tile_sell, kStageCap);
  g.max_sl = p->max_sl;
  g.ns = 2;
  g.cols = p->ngeneric > 0 ? 1 : 0;
  g.npat = p->npat;
  g.poll = owners_poll(p->ntiles) ? 1 : 0;
  g.kib = p->max_ib_row;
  g.ub = p->ub;
  g.red = 0;
  return g;
}

// The chunk sums follow the tile partials in the solve workspace (carve);
// kernels launched with a solve state find them from the partials pointer.
double *chunk_sum_of(const mpb_plan *p, double *part) {
  return part ? reinterpret_cast<double *>(reinterpret_cast<char *>(part) + al256(sizeof(double) * (p->ntiles + 1)))
              : nullptr;
}

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Opt a kernel into the largest dynamic shared memory it may use, once.
// The launch paths never lower the attribute again (probing by setting it
// per candidate size raced with launches from other host threads: an
// in-process slab group launches from one thread per rank).
template <typename K>
void smem_opt_in(K kernel) {
  static std::mutex mu;
  static std::vector<const void *> done;
  std::lock_guard<std::mutex> lk(mu);
  const void *key = reinterpret_cast<const void *>(kernel);
  for (const void *k : done)
    if (k == key) return;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kernel);
  const int mx = optin - static_cast<int>(fa.sharedSizeBytes);
  if (mx > 0) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  done.push_back(key);
}

// Stage count for a persistent tile kernel: the deepest ring (<= kMaxStages)
// that keeps the co-resident CTA count registers and threads allow
// (MPB_STAGES=n forces n; MPB_VERBOSE=1 reports the choice).
template <typename K>
int pick_stages(K kernel, uint32_t stage_bytes, int threads = kWsThreads) {
  auto per_sm = [&](int ns) {
    const uint32_t dyn = ns * stage_bytes;
    if (dyn > 220u * 1024u) return 0;
    smem_opt_in(kernel);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, dyn) != cudaSuccess) n = 0;
    return n;
  };
  static const int forced = std::getenv("MPB_STAGES") ? std::atoi(std::getenv("MPB_STAGES")) : 0;
  const int base = per_sm(2);
  int ns = 2;
  const int cap = forced >= 2 ? std::min(forced, kMaxStages) : 3;
  while (ns < cap && per_sm(ns + 1) >= (forced ? 1 : base)) ns++;
  static const bool verbose = std::getenv("MPB_VERBOSE") != nullptr;
  if (verbose) std::fprintf(stderr, "[mpb] stage %u B: %d stages, %d CTAs/SM\n", stage_bytes, ns, per_sm(ns));
  return ns;
}

// Persistent grid: as many CTAs as are co-resident at this shared-memory
// size, never more than there are tiles.  Opts the kernel into the dynamic
// shared memory it needs.
template <typename K>
int persistent_grid(K kernel, uint32_t dyn_smem, int64_t ntiles, int threads = kCtaThreads) {
  smem_opt_in(kernel);
  static const int carve = std::getenv("MPB_CARVEOUT") ? std::atoi(std::getenv("MPB_CARVEOUT")) : -1;
  if (carve >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn_smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(per_sm) * num_sms())));
}

// Kernel launch, optionally with programmatic stream serialization (PDL):
// the kernel may then start while its predecessor drains, and waits in
// pdl_wait() for the predecessor's results.  Used for the hot kernels of
// the captured single-GPU iteration (MPB_NO_PDL=1 turns it off).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem,
                     cudaStream_t s, Args &&...args) {
  static const bool off = std::getenv("MPB_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && !off) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Buffers one preconditioner application needs besides r and z.
template <typename T>
struct ApplyBufs {
  T *zA, *zB;             // intermediate pass outputs (k > 1)
  T *res, *dg, *wA, *wB;  // large-block path (plan->large)
};

// Tile-claim counter i of the persistent kernels (dynamic scheduling), or
// null for the static walk blockIdx.x, +gridDim.x, ... (MPB_STATIC=1)
unsigned int *claim_ctr(const mpb_handle *h, int i) {
  static const bool stat = std::getenv("MPB_STATIC") && std::atoi(std::getenv("MPB_STATIC")) != 0;
  return stat ? nullptr : h->d_ctr + i;
}

// Warp-per-tile passes (k_bjac_wt / k_update_first_wt) for plans without
// generic rows: an experiment, off by default (MPB_WT=1 turns it on).  On C2
// the last pass took 47 us against 37 us for the CTA-per-tile k_bjac_tile:
// too few warps per SM (two shared-memory stages per warp) for its serial
// eight rows per lane (profiles/r02_notes.md).
bool use_wt() {
  static const bool on = std::getenv("MPB_WT") && std::atoi(std::getenv("MPB_WT")) != 0;
  return on;
}

// Ring depth (stages per consumer warp) of a warp-per-tile kernel: the
// deepest ring up to MPB_WT_DEPTH (default 2) that keeps the resident CTA
// count of the shallowest one.
template <typename K>
int pick_wt_depth(K kernel, uint32_t stage_bytes, int threads) {
  auto per_sm = [&](int depth) {
    const uint32_t dyn = depth * kWtWarps * stage_bytes;
    if (depth * kWtWarps > kWtMaxStages || dyn > 220u * 1024u) return 0;
    smem_opt_in(kernel);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, dyn) != cudaSuccess) n = 0;
    return n;
  };
  static const int forced = std::getenv("MPB_WT_DEPTH") ? std::atoi(std::getenv("MPB_WT_DEPTH")) : 0;
  int depth = 1;
  if (forced > 0) {
    while (depth < forced && per_sm(depth + 1) > 0) depth++;
  } else {  // at least two stages per warp (one in use, one loading), then deeper while the CTA count holds
    if (per_sm(2) > 0) depth = 2;
    const int base = per_sm(depth);
    while (depth < 4 && per_sm(depth + 1) >= base) depth++;
  }
  static const bool verbose = std::getenv("MPB_VERBOSE") != nullptr;
  if (verbose)
    std::fprintf(stderr, "[mpb] wt stage %u B: %d warps x depth %d, %d CTAs/SM\n", stage_bytes, kWtWarps, depth,
                 per_sm(depth));
  return depth;
}

template <typename T, bool F, bool L, bool R64, int KS, bool GEN>
int launch_tile_kernel(mpb_handle *h, cudaStream_t s, const mpb_plan *p, PassArgs<T> a) {
  if (F && !L) {  // first pass streams the in-block layout
    if (a.ib_val == nullptr) return MPB_ERR_LAYOUT;
    a.ib_sp = p->d_ib_sp;
    a.ib_col = p->d_ib_col;
    a.g.cap_e = std::min(p->max_tile_ib, kStageCap);
  }
  const StageLayout Ls = bjac_layout<T, F, R64>(a.g);
  static const bool flat = std::getenv("MPB_FLAT") && std::atoi(std::getenv("MPB_FLAT")) != 0;
  if (!GEN && flat && R64 && !(F && !L) && !a.g.poll) {
    auto kern = k_bjac_flat<T, F, L, KS>;
    MPB_CUDA(launch_k(a.pdl != 0, kern, static_cast<unsigned>(p->ntiles), kTileRows, 0, s, a));
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  if constexpr (!F && !GEN) {
    if (a.win.n > 0 && (reinterpret_cast<uintptr_t>(a.zin) & 15) == 0 && !use_wt()) {
    constexpr int RPT = kLastRpt;
    constexpr int threads = kTileThreads / RPT + 32;
    const StageLayout Lw = bjac_layout_win<T, F, R64>(a.g, a.win);
    auto kern = (L && a.g.poll) ? k_bjac_tile<T, F, L, R64, KS, GEN, L, RPT, true>
                                : k_bjac_tile<T, F, L, R64, KS, GEN, false, RPT, true>;
    a.g.ns = pick_stages(kern, Lw.bytes, threads);
    const uint32_t dyn = a.g.ns * Lw.bytes;
    const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
    MPB_CUDA(launch_k(a.pdl != 0, kern, grid, threads, dyn, s, a));
    MPB_LAUNCHED(h);
    return MPB_OK;
    }
  }
  if (!GEN && use_wt()) {
    constexpr int threads = kWtWarps * 32 + 32;
    auto kern = (L && a.g.poll) ? k_bjac_wt<T, F, L, R64, KS, L> : k_bjac_wt<T, F, L, R64, KS, false>;
    a.g.ns = pick_wt_depth(kern, Ls.bytes, threads) * kWtWarps;
    const uint32_t dyn = a.g.ns * Ls.bytes;
    const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
    MPB_CUDA(launch_k(a.pdl != 0, kern, grid, threads, dyn, s, a));
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  // Offset-slot passes (k_bjac_dia): stencil plans with 64-row blocks
  if constexpr (!F && !GEN && R64 && KS == 7) {
    // (fp64 instances: two fp64 rows per lane need 90 registers; measured against the SELL
    // kernel in the same run, the C3 solve is 0.8 % faster with it; MPB_DIA_F64=0 turns it off)
    static const bool dia64 = !(std::getenv("MPB_DIA_F64") && std::atoi(std::getenv("MPB_DIA_F64")) == 0);
    if (a.dval != nullptr && p->dia_ok && (sizeof(T) == 4 || dia64)) {
      constexpr int threads = kTileThreads / 2 + 32;
      constexpr uint32_t sb = dia_stage_bytes<T>();
      constexpr int kNear = (1 << (kDiaDiag - 1)) | (1 << kDiaDiag) | (1 << (kDiaDiag + 1));
      const bool near = (a.ibany & ~kNear) == 0;  // in-block entries only at the diagonal and its two neighbours
      if (L && a.part != nullptr && a.st != nullptr && red_mode(p)) {  // streamed one-level sum
        a.part = red_part(p, p->n, a.part);
        a.g.red = 1;
      }
      auto kern = near ? ((L && a.g.poll) ? k_bjac_dia<T, L, L, kNear> : k_bjac_dia<T, L, false, kNear>)
                       : ((L && a.g.poll) ? k_bjac_dia<T, L, L, 0x7f> : k_bjac_dia<T, L, false, 0x7f>);
      a.g.ns = pick_stages(kern, sb, threads);
      const uint32_t dyn = a.g.ns * sb;
      const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
      MPB_CUDA(launch_k(a.pdl != 0, kern, grid, threads, dyn, s, a));
      MPB_LAUNCHED(h);
      return MPB_OK;
    }
  }
  // Warp-per-block passes (bjac_tile_wb): plans without generic rows whose
  // blocks all have 64 rows.  Off by default (MPB_WB=1): the same time as the
  // CTA-per-tile kernel on C2 (32.9 us) with 12 % fewer instructions.
  if constexpr (!F && !GEN && R64) {
    static const bool wb_on = std::getenv("MPB_WB") && std::atoi(std::getenv("MPB_WB")) != 0;
    if (wb_on && p->ub == 64 && p->max_ib_row <= 7) {
      constexpr int threads = kTileThreads / 2 + 32;
      auto kern = (L && a.g.poll) ? k_bjac_tile<T, F, L, R64, KS, GEN, L, 2> : k_bjac_tile<T, F, L, R64, KS, GEN, false, 2>;
      a.g.ns = pick_stages(kern, Ls.bytes, threads);
      const uint32_t dyn = a.g.ns * Ls.bytes;
      const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
      MPB_CUDA(launch_k(a.pdl != 0, kern, grid, threads, dyn, s, a));
      MPB_LAUNCHED(h);
      return MPB_OK;
    }
  }
  // the last pass carries the r.z sum: two-level order above MPB_ONE_LEVEL_TILES;
  // a pass that is not the first runs kLastRpt rows per consumer thread
  constexpr int RPT = (!F) ? kLastRpt : kRowsPerThread;
  constexpr int threads = kTileThreads / RPT + 32;
  auto kern = (L && a.g.poll) ? k_bjac_tile<T, F, L, R64, KS, GEN, L, RPT>
                              : k_bjac_tile<T, F, L, R64, KS, GEN, false, RPT>;
  a.g.ns = pick_stages(kern, Ls.bytes, threads);
  const uint32_t dyn = a.g.ns * Ls.bytes;
  const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
  MPB_CUDA(launch_k(a.pdl != 0, kern, grid, threads, dyn, s, a));
  MPB_LAUNCHED(h);
  return MPB_OK;
}

template <typename T, bool F, bool L>
int launch_pass(mpb_handle *h, cudaStream_t s, const mpb_plan *p, PassArgs<T> a, const ApplyBufs<T> &bufs) {
  const int nt = static_cast<int>(p->ntiles);
  if (!p->large) {
    if (p->ks == 7) {
      if (p->ngeneric > 0) {
        if (a.r64 != nullptr) return launch_tile_kernel<T, F, L, true, 7, true>(h, s, p, a);
        return launch_tile_kernel<T, F, L, false, 7, true>(h, s, p, a);
      }
      if (a.r64 != nullptr) return launch_tile_kernel<T, F, L, true, 7, false>(h, s, p, a);
      return launch_tile_kernel<T, F, L, false, 7, false>(h, s, p, a);
    }
    // longer rows (3-T systems): without generic rows the passes that read an fp64
    // residual take the kernels with the full-tile fast path compiled in
    if (a.r64 != nullptr) {
      if (p->ngeneric == 0) return launch_tile_kernel<T, F, L, true, kSlots, false>(h, s, p, a);
      return launch_tile_kernel<T, F, L, true, kSlots, true>(h, s, p, a);
    }
    return launch_tile_kernel<T, F, L, false, kSlots, true>(h, s, p, a);
  }
  a.resbuf = bufs.res;
  a.dbuf = bufs.dg;
  static const bool old_big = std::getenv("MPB_OLD_BIG") != nullptr;
  if (!old_big && p->dia_big && a.dval != nullptr) {
    // offset-slot layout: coalesced slot loads, no pattern-table reads
    const bool pdl = a.pdl != 0;  // chained inside a solve: the next grid is scheduled while this one drains
    MPB_CUDA(launch_k(pdl, k_big_dia_resid<T, F>, static_cast<unsigned>(nt), kCtaThreads, 0, s, a, bufs.wA));
    MPB_LAUNCHED(h);
    T *cur = bufs.wA, *nxt = bufs.wB;
    for (int sweep = 1; sweep < a.t; sweep++) {
      if (sweep + 1 < a.t) {
        MPB_CUDA(launch_k(pdl, k_big_dia_sweep<T, F, L, false>, static_cast<unsigned>(nt), kCtaThreads, 0, s, a,
                          static_cast<const T *>(cur), nxt));
      } else {
        MPB_CUDA(launch_k(pdl, k_big_dia_sweep<T, F, L, true>, static_cast<unsigned>(nt), kCtaThreads, 0, s, a,
                          static_cast<const T *>(cur), nxt));
        MPB_LAUNCHED(h);
        return MPB_OK;
      }
      MPB_LAUNCHED(h);
      std::swap(cur, nxt);
    }
    k_big_finish<T, F, L><<<nt, kCtaThreads, 0, s>>>(a, cur);  // t == 1: no sweep to carry the finish
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  if (!old_big && a.meta != nullptr && a.pat != nullptr && p->npat > 0) {
    // row patterns: no column stream, no block search, finish fused into the last sweep
    k_big_resid_pat<T, F><<<nt, kCtaThreads, 0, s>>>(a, bufs.wA);
    MPB_LAUNCHED(h);
    T *cur = bufs.wA, *nxt = bufs.wB;
    for (int sweep = 1; sweep < a.t; sweep++) {
      if (sweep + 1 < a.t) {
        k_big_sweep_pat<T, F, L, false><<<nt, kCtaThreads, 0, s>>>(a, cur, nxt);
      } else {
        k_big_sweep_pat<T, F, L, true><<<nt, kCtaThreads, 0, s>>>(a, cur, nxt);
        MPB_LAUNCHED(h);
        return MPB_OK;
      }
      MPB_LAUNCHED(h);
      std::swap(cur, nxt);
    }
    k_big_finish<T, F, L><<<nt, kCtaThreads, 0, s>>>(a, cur);  // t == 1: no sweep to carry the finish
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  k_big_resid<T, F><<<nt, kCtaThreads, 0, s>>>(a, bufs.wA);
  MPB_LAUNCHED(h);
  T *cur = bufs.wA, *nxt = bufs.wB;
  for (int sweep = 1; sweep < a.t; sweep++) {
    k_big_sweep<T><<<nt, kCtaThreads, 0, s>>>(a, cur, nxt);
    MPB_LAUNCHED(h);
    std::swap(cur, nxt);
  }
  k_big_finish<T, F, L><<<nt, kCtaThreads, 0, s>>>(a, cur);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

// the operator of the outer SpMV and the true residuals (solver.py:154, 93-98)
static const double *op_vals(const mpb_csr *A) { return A->op_sell_val64 ? A->op_sell_val64 : A->sell_val64; }

template <typename T>
const T *sell_vals(const mpb_csr *A);
template <>
const double *sell_vals<double>(const mpb_csr *A) {
  return A->sell_val64;
}
template <>
const float *sell_vals<float>(const mpb_csr *A) {
  return A->sell_val32;
}
template <typename T>
const T *ib_vals(const mpb_csr *A);
template <>
const double *ib_vals<double>(const mpb_csr *A) {
  return A->ib_val64;
}
template <>
const float *ib_vals<float>(const mpb_csr *A) {
  return A->ib_val32;
}

// k outer passes (bjac.py:127-149).  Residual from r64 (narrowed on load) or
// rT; final output to zout (T) and/or zout64; r.z partials when part != null
// (and, in solve mode, the fused rho step in the last CTA).
// multi-GPU context of a solve (null on one GPU)
struct DistCtx {
  const mpb_comm *comm;
  mpb_halo halo;
};

// In-process group: rank 0 copies every rank's ghost rows from its
// neighbours' own rows (what the NCCL path sends and receives).
int local_halo(const DistCtx *dc, void *buf, int es, int64_t n, cudaStream_t s) {
  LocalGroup &G = *dc->comm->grp;
  const int me = dc->comm->rank;
  G.slot[me].buf = buf;
  G.slot[me].es = es;
  G.slot[me].n = n;
  G.slot[me].halo = dc->halo;
  if (!G.barrier(me, "halo-in")) return MPB_ERR_COMM;
  int rc = MPB_OK;
  if (me == 0) {
    for (int r = 0; r < G.nranks && rc == MPB_OK; r++) {
      const LocalGroup::Slot &R = G.slot[r];
      char *dst = static_cast<char *>(R.buf) + R.n * es;
      if (R.halo.rank_lo >= 0 && R.halo.recv_lo > 0) {  // rows just below: the lower rank's top rows
        const LocalGroup::Slot &L = G.slot[R.halo.rank_lo];
        if (cudaMemcpyAsync(dst, static_cast<const char *>(L.buf) + (L.n - R.halo.recv_lo) * es, R.halo.recv_lo * es,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
          rc = MPB_ERR_COMM;
      }
      if (R.halo.rank_hi >= 0 && R.halo.recv_hi > 0) {  // rows just above: the upper rank's first rows
        const LocalGroup::Slot &U = G.slot[R.halo.rank_hi];
        if (cudaMemcpyAsync(dst + R.halo.recv_lo * es, U.buf, R.halo.recv_hi * es, cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess)
          rc = MPB_ERR_COMM;
      }
    }
  }
  if (!G.barrier(me, "halo-out")) return MPB_ERR_COMM;
  return rc;
}

// Fill the ghost rows [n, n+ng) of `buf` from the neighbouring slabs and
// send ours (NCCL grouped point-to-point, on the solve stream).
int halo_exchange(const DistCtx *dc, void *buf, int es, int64_t n, cudaStream_t s) {
  if (dc == nullptr) return MPB_OK;
  if (dc->comm->grp != nullptr) return local_halo(dc, buf, es, n, s);
  NcclApi &N = nccl();
  const mpb_halo &hl = dc->halo;
  const int dt = es == 8 ? kNcclFloat64 : kNcclFloat32;
  char *b = static_cast<char *>(buf);
  if (N.GroupStart() != 0) return MPB_ERR_COMM;
  int e = 0;
  if (hl.rank_lo >= 0) {
    if (hl.send_lo > 0) e |= N.Send(b, hl.send_lo, dt, hl.rank_lo, dc->comm->comm, s);
    if (hl.recv_lo > 0) e |= N.Recv(b + n * es, hl.recv_lo, dt, hl.rank_lo, dc->comm->comm, s);
  }
  if (hl.rank_hi >= 0) {
    if (hl.send_hi > 0) e |= N.Send(b + (n - hl.send_hi) * es, hl.send_hi, dt, hl.rank_hi, dc->comm->comm, s);
    if (hl.recv_hi > 0) e |= N.Recv(b + (n + hl.recv_lo) * es, hl.recv_hi, dt, hl.rank_hi, dc->comm->comm, s);
  }
  e |= N.GroupEnd();
  return e ? MPB_ERR_COMM : MPB_OK;
}

// Multi-GPU scalar step: all-reduce this rank's sum, then run the step.
int dist_step(mpb_handle *h, const DistCtx *dc, SolverState *st, int step, int gate, cudaStream_t s) {
  if (dc == nullptr) return MPB_OK;
  if (dc->comm->grp != nullptr) {  // in-process group: rank-ordered sum of the ranks' partials
    LocalGroup &G = *dc->comm->grp;
    const int me = dc->comm->rank;
    G.slot[me].st = st;
    if (!G.barrier(me, "step-in")) return MPB_ERR_COMM;
    int rc = MPB_OK;
    if (me == 0) {  // the states travel as kernel arguments (no host-to-device copy)
      LocalStates sts{};
      for (int r = 0; r < G.nranks; r++) sts.p[r] = G.slot[r].st;
      k_local_allreduce<<<1, 32, 0, s>>>(sts, G.nranks);
      MPB_LAUNCHED(h);
    }
    if (!G.barrier(me, "step-out")) return MPB_ERR_COMM;
    if (rc) return rc;
    k_apply_step<<<1, 32, 0, s>>>(step, st, gate);
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  NcclApi &N = nccl();
  if (N.AllReduce(st->red_local, st->red_global, 2, kNcclFloat64, kNcclSum, dc->comm->comm, s) != 0)
    return MPB_ERR_COMM;
  k_apply_step<<<1, 32, 0, s>>>(step, st, gate);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

// the plan's offset-slot layout (the values follow the in-block values in
// the plan-packed buffer a.ib_val)
template <typename T>
void bind_dia(PassArgs<T> &a, const mpb_plan *p) {
  if (!p->dia_layout || a.ib_val == nullptr) return;
  a.dval = a.ib_val + p->dia_at;
  a.dnear = p->near_entries > 0 ? a.ib_val + p->near_at : nullptr;
  a.dmeta = p->d_dmeta;
  for (int u = 0; u < kDiaSlots; u++) a.doff[u] = p->dia_off[u];
  a.ibany = p->dia_ibany;
}

template <typename T>
int launch_apply(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const mpb_csr *A, int k, int t,
                 const double *r64, const T *rT, T *zout, double *zout64, double *part,
                 unsigned long long *ovf_count, long long *ovf_first, SolverState *st, int want_branch,
                 const ApplyBufs<T> &bufs, const DistCtx *dc = nullptr, int from_pass = 0, int to_pass = 1 << 30,
                 int z1_gate = 0, int prefetch = 0) {
  PassArgs<T> a{};
  a.sp = A->sell->d_sp;
  a.scol = A->sell->d_col;
  a.sval = sell_vals<T>(A);
  a.ib_val = ib_vals<T>(A);
  a.meta = p->d_meta;
  a.pat = p->d_pat;
  a.td = p->d_td;
  a.ctr = claim_ctr(h, 0);
  a.boff = p->d_boff;
  a.g = geom_for<T>(p);
  a.t = t;
  a.r64 = r64;
  a.rT = rT;
  a.ovf_count = ovf_count;
  a.ovf_first = ovf_first;
  a.st = st;
  a.csum = st ? chunk_sum_of(p, part) : nullptr;
  a.want_branch = want_branch;
  a.pdl = (st != nullptr && dc == nullptr) ? 1 : 0;  // captured single-GPU iteration
  a.gate = z1_gate;
  a.prefetch = prefetch;
  if (dc == nullptr) {  // gather windows: one GPU (slabs' ghost columns are not row + offset)
    a.win = p->win;
    a.win.zlen = static_cast<int>(A->n);
  }
  bind_dia(a, p);
  for (int pass = from_pass; pass < std::min(k, to_pass); pass++) {
    const bool first = pass == 0, last = pass == k - 1;
    a.zin = first ? nullptr : ((pass - 1) & 1 ? bufs.zB : bufs.zA);
    a.zout = last ? zout : (pass & 1 ? bufs.zB : bufs.zA);
    a.zout64 = last ? zout64 : nullptr;
    a.part = last ? part : nullptr;
    int rc;
    if (first && last) rc = launch_pass<T, true, true>(h, s, p, a, bufs);
    else if (first) rc = launch_pass<T, true, false>(h, s, p, a, bufs);
    else if (last) rc = launch_pass<T, false, true>(h, s, p, a, bufs);
    else rc = launch_pass<T, false, false>(h, s, p, a, bufs);
    if (rc) return rc;
    if (!last) {  // the next pass gathers this pass's output across slabs
      rc = halo_exchange(dc, a.zout, sizeof(T), A->n, s);
      if (rc) return rc;
    }
  }
  return MPB_OK;
}

// The fused x/r update + next first pass (k_update_first) of one branch.
template <typename T>
int launch_update_first(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const mpb_csr *A, int t, T *z1,
                        double *x, const double *pv, const double *q, double *r, double *part,
                        unsigned long long *ovf_count, long long *ovf_first, SolverState *st, int want_branch,
                        int prefetch = 0, bool pdl = true) {
  PassArgs<T> a{};
  a.sp = A->sell->d_sp;
  a.scol = A->sell->d_col;
  a.sval = sell_vals<T>(A);
  a.ib_val = ib_vals<T>(A);
  a.ib_sp = p->d_ib_sp;
  a.ib_col = p->d_ib_col;
  if (a.ib_val == nullptr) return MPB_ERR_LAYOUT;
  a.meta = p->d_meta;
  a.pat = p->d_pat;
  a.td = p->d_td;
  a.ctr = claim_ctr(h, 1);
  a.boff = p->d_boff;
  a.g = geom_for<T>(p);
  a.g.cap_e = std::min(p->max_tile_ib, kStageCap);
  a.t = t;
  a.zout = z1;
  a.part = part;
  a.ovf_count = ovf_count;
  a.ovf_first = ovf_first;
  a.st = st;
  a.csum = st ? chunk_sum_of(p, part) : nullptr;
  a.want_branch = want_branch;
  a.gate = 2;
  a.prefetch = prefetch;
  bind_dia(a, p);
  if (a.dnear != nullptr && a.part != nullptr && st != nullptr) {  // offset-slot layout, warp per block
    constexpr int threads = kTileThreads / 2 + 32;
    constexpr uint32_t sb = dia_uf_stage_bytes<T>();
    if (red_mode(p)) {  // streamed one-level sum
      a.part = red_part(p, p->n, a.part);
      a.g.red = 1;
    }
    auto kern = two_level(p->ntiles) ? k_update_first_dia<T, true> : k_update_first_dia<T, false>;
    a.g.ns = pick_stages(kern, sb, threads);
    const uint32_t dyn = a.g.ns * sb;
    const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
    MPB_CUDA(launch_k(pdl, kern, grid, threads, dyn, s, a, x, pv, q, r));
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  const StageLayout L = update_first_layout<T>(a.g);
  if (p->ngeneric == 0 && use_wt()) {
    constexpr int threads = kWtWarps * 32 + 32;
    auto kern = two_level(p->ntiles) ? k_update_first_wt<T, true> : k_update_first_wt<T, false>;
    a.g.ns = pick_wt_depth(kern, L.bytes, threads) * kWtWarps;
    const uint32_t dyn = a.g.ns * L.bytes;
    const int grid = persistent_grid(kern, dyn, p->ntiles, threads);
    MPB_CUDA(launch_k(pdl, kern, grid, threads, dyn, s, a, x, pv, q, r));
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  auto kern = two_level(p->ntiles) ? (p->ngeneric > 0 ? k_update_first_two<T, true> : k_update_first_two<T, false>)
                                    : (p->ngeneric > 0 ? k_update_first<T, true> : k_update_first<T, false>);
  a.g.ns = pick_stages(kern, L.bytes);
  const uint32_t dyn = a.g.ns * L.bytes;
  const int grid = persistent_grid(kern, dyn, p->ntiles, kWsThreads);
  MPB_CUDA(launch_k(pdl, kern, grid, kWsThreads, dyn, s, a, x, pv, q, r));
  MPB_LAUNCHED(h);
  return MPB_OK;
}

// The wave kernel (k_wave) of one fixed branch: x/r update + first pass of
// iteration i and the last pass of iteration i+1.  z1: the first pass's
// output (the last pass's z_in); zout: the last pass's output.
template <typename T>
int launch_wave(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const mpb_csr *A, int t, T *z1, T *zout,
                double *x, const double *pv, const double *q, double *r, double *part_rr, double *part_rz,
                unsigned int *gcnt, unsigned long long *ovf_count, long long *ovf_first, SolverState *st,
                int want_branch, bool pdl = true) {
  if (!p->wave_ok) return MPB_ERR_LAYOUT;
  PassArgs<T> au{};
  au.sp = A->sell->d_sp;
  au.sval = sell_vals<T>(A);
  au.ib_val = ib_vals<T>(A);
  au.ib_sp = p->d_ib_sp;
  au.ib_col = p->d_ib_col;
  if (au.ib_val == nullptr || au.sval == nullptr) return MPB_ERR_LAYOUT;
  au.meta = p->d_meta;
  au.pat = p->d_pat;
  au.td = p->d_td;
  au.ctr = claim_ctr(h, 1);
  au.boff = p->d_boff;
  au.g = geom_for<T>(p);
  au.g.cap_e = p->max_tile_ib;
  au.t = t;
  au.zout = z1;
  au.part = part_rr;
  au.ovf_count = ovf_count;
  au.ovf_first = ovf_first;
  au.st = st;
  au.want_branch = want_branch;
  au.gate = 2;
  PassArgs<T> al = au;
  al.ib_sp = nullptr;
  al.ib_col = nullptr;
  al.ib_val = nullptr;
  al.g = geom_for<T>(p);
  al.g.cap_e = static_cast<int>(p->max_tile_sell);
  al.r64 = r;
  al.zin = z1;
  al.zout = zout;
  al.part = part_rz;
  al.ovf_count = nullptr;
  al.ovf_first = nullptr;
  const uint32_t sb = std::max(update_first_layout<T>(au.g).bytes,
                               stage_layout(al.g.cap_e, sizeof(T), al.g.max_sl, false, true, 0, 0, 0).bytes);
  void (*kern)(const PassArgs<T>, const PassArgs<T>, double *, const double *, const double *, double *,
               const WaveCtl) = nullptr;
  if (p->ks == 7) kern = p->max_ib_row <= 3 ? k_wave<T, 7, 3> : k_wave<T, 7, 7>;
  else kern = k_wave<T, kSlots, 7>;
  au.g.ns = al.g.ns = pick_stages(kern, sb, kTileThreads + 32);
  const uint32_t dyn = au.g.ns * sb;
  const int grid = persistent_grid(kern, dyn, 2 * p->ntiles, kTileThreads + 32);
  static const int dbg = std::getenv("MPB_WAVE_DBG") ? std::atoi(std::getenv("MPB_WAVE_DBG")) : 0;
  const WaveCtl wc{gcnt, p->d_wdep, p->wave_lag, p->wave_gshift, dbg, static_cast<int>(p->ntiles / 32 + 4)};
  MPB_CUDA(launch_k(pdl, kern, grid, kTileThreads + 32, dyn, s, au, al, x, pv, q, r, wc));
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int check_csr(const mpb_csr *A) {
  if (!A || !A->row_ptr || !A->col_idx || A->n < 1) return MPB_ERR_ARG;
  if (A->n >= (int64_t(1) << 31) - 1 || A->nnz >= (int64_t(1) << 31)) return MPB_ERR_INDEX32;
  return MPB_OK;
}

// hot entry points read the SELL-32 layout
int check_bound(const mpb_plan *p, const mpb_csr *A) {
  return (p != nullptr && A != nullptr && p->d_meta != nullptr && p->bound == A->sell) ? MPB_OK : MPB_ERR_LAYOUT;
}

int check_sell(const mpb_csr *A, bool need64, bool need32) {
  int rc = check_csr(A);
  if (rc) return rc;
  if (!A->sell || A->sell->n != A->n) return MPB_ERR_LAYOUT;
  if (need64 && !A->sell_val64) return MPB_ERR_LAYOUT;
  if (need32 && !A->sell_val32) return MPB_ERR_LAYOUT;
  return MPB_OK;
}

// partition/tile plan, same rule as include/mpbjac_order.h (and the oracle)
int64_t plan_tiles(int64_t nb, const int64_t *offs, const int64_t *rp, int64_t *tile_lo, int *large) {
  int64_t nt = 0, cur_lo = 0, cur_rows = 0, cur_nnz = 0;
  *large = 0;
  for (int64_t b = 0; b < nb; b++) {
    const int64_t lo = offs[b], hi = offs[b + 1];
    const int64_t br = hi - lo, bz = rp[hi] - rp[lo];
    if (br > MPB_TILE_MAX_ROWS) {
      if (cur_rows > 0) tile_lo[nt++] = cur_lo;
      for (int64_t s = lo; s < hi; s += MPB_TILE_MAX_ROWS) tile_lo[nt++] = s;
      cur_lo = hi;
      cur_rows = cur_nnz = 0;
      *large = 1;
      continue;
    }
    if (cur_rows > 0 && (cur_rows + br > MPB_TILE_MAX_ROWS || cur_nnz + bz > MPB_TILE_PACK_NNZ)) {
      tile_lo[nt++] = cur_lo;
      cur_lo = lo;
      cur_rows = cur_nnz = 0;
    }
    cur_rows += br;
    cur_nnz += bz;
  }
  if (cur_rows > 0) tile_lo[nt++] = cur_lo;
  tile_lo[nt] = offs[nb];
  return nt;
}

// Solve-time workspace layout
struct SolveWs {
  double *r, *q, *p, *p2, *z64, *zA64, *zB64;  // p2: second search-direction buffer (fused mode)
  float *z32, *zA32, *zB32;
  double *res64, *dg64, *wA64, *wB64;
  float *res32, *dg32, *wA32, *wB32;
  double *part;
  double *part2;       // wave kernel: the r.z tile partials of its last-pass items (part: r.r)
  double *part3;       // k_solve_small: one array per dot product (part r.z, part2 p.q, part3 r.r)
  double *ppart;       // streamed one-level sums of the offset-slot kernels (red_mode)
  unsigned int *gcnt;  // wave kernel: per tile group, update items published this solve
  double *csum;        // chunk sums of the two-level dot sums (part: all slots kPartEmpty between kernels)
  SolverState *st;
  size_t bytes;
};

// ng: ghost rows of a multi-GPU slab (0 on one GPU); vectors that kernels
// gather from (p, pass outputs) carry them after the n own rows
SolveWs carve(const mpb_plan *p, int64_t n, char *base, int64_t ng = 0) {
  SolveWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) -> char * {
    char *q = base ? base + off : nullptr;
    off += al256(bytes);
    return q;
  };
  const size_t d = sizeof(double) * (n + 2), f = sizeof(float) * (n + 4);
  const size_t dg = sizeof(double) * (n + ng + 2), fg = sizeof(float) * (n + ng + 4);
  w.r = (double *)take(d);
  w.q = (double *)take(d);
  w.p = (double *)take(dg);
  w.p2 = (double *)take(dg);
  w.z64 = (double *)take(dg);
  w.zA64 = (double *)take(dg);
  w.zB64 = (double *)take(dg);
  w.z32 = (float *)take(fg);
  w.zA32 = (float *)take(fg);
  w.zB32 = (float *)take(fg);
  if (p->large) {
    w.res64 = (double *)take(d);
    w.dg64 = (double *)take(d);
    w.wA64 = (double *)take(d);
    w.wB64 = (double *)take(d);
    w.res32 = (float *)take(f);
    w.dg32 = (float *)take(f);
    w.wA32 = (float *)take(f);
    w.wB32 = (float *)take(f);
  }
  w.part = (double *)take(sizeof(double) * (p->ntiles + 1));
  w.part2 = (double *)take(sizeof(double) * (p->ntiles + 1));
  w.part3 = (double *)take(sizeof(double) * (p->ntiles + 1));
  w.gcnt = (unsigned int *)take(sizeof(unsigned int) * (p->ntiles / 32 + 8));
  w.csum = (double *)take(sizeof(double) * ((p->ntiles + kChunkTiles - 1) / kChunkTiles + 1));
  // streamed one-level sums (reduce_stream): their own tile partials, all slots kPartEmpty between kernels
  w.ppart = (double *)take(sizeof(double) * (p->ntiles + 1));
  w.st = (SolverState *)take(sizeof(SolverState));
  w.bytes = off;
  return w;
}

// Streamed one-level sums (reduce_stream) for the offset-slot kernels: plans
// of 64 to 8,192 tiles (above, the two-level order has its chunk owners).
// MPB_RED=0 turns it off.
// The kernels get their own partials array (every slot kPartEmpty between
// kernels), found from the solve's partials pointer (carve's layout).
bool red_mode(const mpb_plan *p) {
  // (the static tile walk of MPB_STATIC=1 assumes every CTA takes tiles)
  static const bool off = (std::getenv("MPB_RED") && std::atoi(std::getenv("MPB_RED")) == 0) ||
                          (std::getenv("MPB_STATIC") && std::atoi(std::getenv("MPB_STATIC")) != 0);
  return !off && p->dia_ok && !two_level(p->ntiles) && p->ntiles >= 64;  // (CTA 0 takes no tiles: the grid needs more)
}
double *red_part(const mpb_plan *p, int64_t n, double *part) {
  char *const fake = reinterpret_cast<char *>(uintptr_t(1) << 20);
  const SolveWs f = carve(p, n, fake);
  return reinterpret_cast<double *>(reinterpret_cast<char *>(part) +
                                    (reinterpret_cast<char *>(f.ppart) - reinterpret_cast<char *>(f.part)));
}



}  // namespace

// ===========================================================================
// C-ABI (C linkage comes from the declarations in include/mpbjac.h)
// ===========================================================================

int mpb_version(void) { return MPB_VERSION; }

const char *mpb_status_string(int status) {
  switch (status) {
    case MPB_OK: return "ok";
    case MPB_ERR_ARG: return "invalid argument";
    case MPB_ERR_SHAPE: return "inconsistent shapes";
    case MPB_ERR_PARTITION: return "partition does not match the matrix";
    case MPB_ERR_SWEEPS: return "sweep counts k and t must be at least 1";
    case MPB_ERR_INDEX32: return "matrix too large for int32 indexing";
    case MPB_ERR_POLICY: return "policy needs a preconditioner instance that was not set up";
    case MPB_ERR_WORKSPACE: return "workspace too small";
    case MPB_ERR_LAYOUT: return "matrix has no SELL-32 layout (mpb_sell_create / mpb_sell_pack_*)";
    case MPB_ERR_COMM: return "NCCL unavailable or a collective failed";
    default: break;
  }
  if (status > 0) return cudaGetErrorString(static_cast<cudaError_t>(status));
  return "unknown status";
}

int mpb_create(int device, void *stream, mpb_handle **out) {
  if (!out) return MPB_ERR_ARG;
  *out = nullptr;
  MPB_CUDA(cudaSetDevice(device));
  mpb_handle *h = new mpb_handle();
  h->device = device;
  h->user = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaStreamCreateWithFlags(&h->solve, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev_t0);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev_t1);
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_state, sizeof(SolverState));
  if (e == cudaSuccess) e = cudaMalloc(&h->d_ctr, 16 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(h->d_ctr, 0, 16 * sizeof(unsigned int));
  if (e != cudaSuccess) {
    delete h;
    return status_of(e);
  }
  *out = h;
  return MPB_OK;
}

int mpb_destroy(mpb_handle *h) {
  if (!h) return MPB_OK;
  cudaStreamSynchronize(h->user);
  cudaStreamSynchronize(h->solve);
  if (h->have_graph) cudaGraphExecDestroy(h->gexec);
  if (h->scratch) cudaFree(h->scratch);
  cudaFreeHost(h->h_state);
  cudaFree(h->d_ctr);
  cudaFree(h->d_tl);
  cudaEventDestroy(h->ev_in);
  cudaEventDestroy(h->ev_out);
  cudaEventDestroy(h->ev_t0);
  cudaEventDestroy(h->ev_t1);
  cudaStreamDestroy(h->solve);
  delete h;
  cudaGetLastError();  // (a user stream destroyed first must not leave a stale error behind)
  return MPB_OK;
}

int mpb_set_stream(mpb_handle *h, void *stream) {
  if (!h) return MPB_ERR_ARG;
  h->user = static_cast<cudaStream_t>(stream);
  return MPB_OK;
}

int mpb_synchronize(mpb_handle *h) {
  if (!h) return MPB_ERR_ARG;
  MPB_CUDA(cudaStreamSynchronize(h->user));
  MPB_CUDA(cudaStreamSynchronize(h->solve));
  return MPB_OK;
}

int64_t mpb_launch_count(const mpb_handle *h) { return h ? h->launches : 0; }

// ---- plans -----------------------------------------------------------------
int64_t mpb_plan_tiles_host(int64_t nb, const int64_t *h_offsets, const int64_t *h_row_ptr, int64_t *h_tile_lo,
                            int *h_large) {
  if (nb < 1 || !h_offsets || !h_row_ptr || !h_tile_lo || !h_large) return MPB_ERR_ARG;
  return plan_tiles(nb, h_offsets, h_row_ptr, h_tile_lo, h_large);
}

int mpb_plan_create(mpb_handle *h, int64_t n, int64_t nb, const int64_t *h_offsets, const int64_t *h_row_ptr,
                    mpb_plan **out) {
  if (!h || !out || !h_offsets || !h_row_ptr || nb < 1 || n < 1) return MPB_ERR_ARG;
  *out = nullptr;
  if (h_offsets[0] != 0 || h_offsets[nb] != n) return MPB_ERR_PARTITION;
  for (int64_t b = 0; b < nb; b++)
    if (h_offsets[b + 1] <= h_offsets[b]) return MPB_ERR_PARTITION;
  if (n >= (int64_t(1) << 31) - 1 || h_row_ptr[n] >= (int64_t(1) << 31)) return MPB_ERR_INDEX32;
  std::vector<int64_t> tlo(nb + n / MPB_TILE_MAX_ROWS + 2);
  int large = 0;
  const int64_t nt = plan_tiles(nb, h_offsets, h_row_ptr, tlo.data(), &large);
  std::vector<int> tl(nt + 1), bfv(nt), blv(nt), boff(nb + 1);
  int64_t max_nnz = 0;
  int64_t b = 0;
  for (int64_t i = 0; i <= nt; i++) tl[i] = static_cast<int>(tlo[i]);
  for (int64_t i = 0; i <= nb; i++) boff[i] = static_cast<int>(h_offsets[i]);
  for (int64_t i = 0; i < nt; i++) {
    const int64_t lo = tlo[i], hi = tlo[i + 1];
    while (h_offsets[b + 1] <= lo) b++;
    bfv[i] = static_cast<int>(b);
    int64_t e = b;
    while (h_offsets[e + 1] < hi) e++;
    blv[i] = static_cast<int>(e);
    max_nnz = std::max(max_nnz, h_row_ptr[hi] - h_row_ptr[lo]);
  }
  // tile descriptors against the SELL-32 slice layout of this structure
  std::vector<int> sp;
  if (!sell_slice_ptrs(n, h_row_ptr, sp)) return MPB_ERR_INDEX32;
  std::vector<TileDesc> td(nt);
  int max_sell = 0, max_sl = 0, max_nbk = 0;
  for (int64_t i = 0; i < nt; i++) {
    TileDesc &d = td[i];
    d.lo = tl[i];
    d.hi = tl[i + 1];
    d.s0 = d.lo >> 5;
    d.s1 = (d.hi + 31) >> 5;
    d.e0 = sp[d.s0];
    d.e1 = sp[d.s1];
    d.bf = bfv[i];
    d.nbk = blv[i] - bfv[i] + 1;
    max_sell = std::max(max_sell, d.e1 - d.e0);
    max_sl = std::max(max_sl, d.s1 - d.s0);
    max_nbk = std::max(max_nbk, d.nbk);
  }
  MPB_CUDA(cudaSetDevice(h->device));
  mpb_plan *p = new mpb_plan();
  p->device = h->device;
  p->n = n;
  p->nb = nb;
  p->ntiles = nt;
  p->large = large;
  p->max_tile_nnz = max_nnz;
  p->max_tile_sell = max_sell;
  p->max_sl = max_sl;
  p->max_nbk = max_nbk;
  p->ub = static_cast<int>(h_offsets[1] - h_offsets[0]);
  for (int64_t i = 1; i < nb && p->ub != 0; i++)
    if (h_offsets[i + 1] - h_offsets[i] != p->ub) p->ub = 0;
  cudaError_t e = cudaMalloc(&p->d_tile_lo, sizeof(int) * (nt + 1));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_tile_bf, sizeof(int) * nt);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_tile_bl, sizeof(int) * nt);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_boff, sizeof(int) * (nb + 1));
  if (e == cudaSuccess) e = cudaMemcpy(p->d_tile_lo, tl.data(), sizeof(int) * (nt + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_tile_bf, bfv.data(), sizeof(int) * nt, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_tile_bl, blv.data(), sizeof(int) * nt, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_boff, boff.data(), sizeof(int) * (nb + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_td, sizeof(TileDesc) * nt);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_td, td.data(), sizeof(TileDesc) * nt, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    mpb_plan_destroy(p);
    return status_of(e);
  }
  *out = p;
  return MPB_OK;
}

int mpb_plan_destroy(mpb_plan *p) {
  if (!p) return MPB_OK;
  cudaFree(p->d_tile_lo);
  cudaFree(p->d_tile_bf);
  cudaFree(p->d_tile_bl);
  cudaFree(p->d_boff);
  cudaFree(p->d_td);
  cudaFree(p->d_meta);
  cudaFree(p->d_ib_sp);
  cudaFree(p->d_ib_col);
  cudaFree(p->d_pmask);
  cudaFree(p->d_U);
  cudaFree(p->d_wdep);
  cudaFree(p->d_dmeta);
  cudaFree(p->d_pslot);
  delete p;
  return MPB_OK;
}

// Wave kernel eligibility and dependencies (k_wave): pattern rows only,
// every tile a multiple of 32 rows at a 32-row-aligned start (the full-tile
// bodies), stages that hold every tile, one-level sums.  A tile's last pass
// reads rows [lo + omin, hi - 1 + omax] (the patterns' extreme offsets); its
// dependency range is the tile groups covering them, and the item lag
// exceeds the farthest tile such a group reaches (plus slack for the items
// in flight, MPB_WAVE_SLACK, default 1536 tiles).  Off by default (MPB_WAVE=1
// enables it): on C2 the wave kernel takes 67.1 us against 64.5 us for the
// last pass + fused update it replaces -- each publication's gpu-scope
// release (MEMBAR.ALL.GPU) costs the SM more than the kernel boundary it
// saves (61.2 us with an unfenced, unsafe publication; profiles/r02_notes.md).
static int plan_wave(mpb_handle *h, mpb_plan *p, const std::vector<TileDesc> &td) {
  p->wave_ok = false;
  static const bool off = !(std::getenv("MPB_WAVE") && std::atoi(std::getenv("MPB_WAVE")) != 0);
  if (off || p->large || p->ngeneric != 0 || p->npat <= 0 || two_level(p->ntiles) || p->max_ib_row > 7 ||
      p->max_tile_sell > kStageCap || p->max_tile_ib > kStageCap)
    return MPB_OK;
  for (const auto &d : td)
    if ((d.lo & 31) != 0 || ((d.hi - d.lo) & 31) != 0) return MPB_OK;
  std::vector<int> pat(static_cast<size_t>(p->npat) * kPatStride);
  MPB_CUDA(cudaMemcpy(pat.data(), p->d_pat, sizeof(int) * pat.size(), cudaMemcpyDeviceToHost));
  int omin = 0, omax = 0;
  for (int q = 0; q < p->npat; q++) {
    const int *P = &pat[static_cast<size_t>(q) * kPatStride];
    for (int u = 0; u < (P[0] & 0xFF); u++) {
      omin = std::min(omin, P[1 + u]);
      omax = std::max(omax, P[1 + u]);
    }
  }
  const int64_t nt = p->ntiles, n = p->n;
  const int gs = p->wave_gshift;
  std::vector<int> lo(nt);
  for (int64_t i = 0; i < nt; i++) lo[i] = td[i].lo;
  auto tile_of = [&](int64_t row) {
    return static_cast<int>(std::upper_bound(lo.begin(), lo.end(), static_cast<int>(row)) - lo.begin()) - 1;
  };
  std::vector<int2> dep(nt);
  int64_t reach = 0;
  for (int64_t i = 0; i < nt; i++) {
    const int t0 = tile_of(std::max<int64_t>(0, td[i].lo + int64_t(omin)));
    const int t1 = tile_of(std::min<int64_t>(n - 1, td[i].hi - 1 + int64_t(omax)));
    dep[i] = make_int2(t0 >> gs, t1 >> gs);
    const int64_t far = std::min<int64_t>(nt - 1, ((int64_t(t1 >> gs) + 1) << gs) - 1);
    reach = std::max(reach, far - i);
  }
  static const int slack = std::getenv("MPB_WAVE_SLACK") ? std::atoi(std::getenv("MPB_WAVE_SLACK")) : 1536;
  p->wave_lag = static_cast<int>(std::min<int64_t>(nt, reach + 1 + std::max(slack, 0)));
  p->wave_ngroups = static_cast<int>((nt + (1 << gs) - 1) >> gs);
  cudaFree(p->d_wdep);
  p->d_wdep = nullptr;
  MPB_CUDA(cudaMalloc(&p->d_wdep, sizeof(int2) * nt));
  MPB_CUDA(cudaMemcpy(p->d_wdep, dep.data(), sizeof(int2) * nt, cudaMemcpyHostToDevice));
  p->wave_ok = true;
  if (std::getenv("MPB_VERBOSE"))
    std::fprintf(stderr, "[mpb] wave: offsets [%d, %d], reach %lld tiles, lag %d of %lld tiles, %d groups\n", omin,
                 omax, static_cast<long long>(reach), p->wave_lag, static_cast<long long>(nt), p->wave_ngroups);
  (void)h;
  return MPB_OK;
}

// Offset-slot layout (k_bjac_dia) for a plan bound to its SELL structure:
// eligible when every row has a pattern, the patterns' column offsets are
// drawn from exactly kDiaSlots values with 0 in the middle (a 7-point
// stencil in any grid size), and every block has 64 rows.  MPB_DIA=0 turns
// it off (the SELL kernels then run).
static int plan_dia(mpb_handle *h, mpb_plan *p) {
  p->dia_layout = p->dia_ok = p->dia_big = false;
  p->dia_entries = 0;
  p->dia_at = 0;
  p->near_entries = 0;
  static const bool off = std::getenv("MPB_DIA") && std::atoi(std::getenv("MPB_DIA")) == 0;
  if (off || p->ngeneric != 0 || p->npat <= 0 || p->max_ib_row > kDiaSlots) return MPB_OK;
  if (!p->large && p->ub != 64) return MPB_OK;  // (tile kernels: a warp per 64-row block)
  if (p->large) {  // every row must have row metadata (large plans do not count generic rows per tile)
    static const bool big_off = std::getenv("MPB_DIA_BIG") && std::atoi(std::getenv("MPB_DIA_BIG")) == 0;
    if (big_off) return MPB_OK;
    std::vector<uint16_t> meta(p->n);
    MPB_CUDA(cudaMemcpy(meta.data(), p->d_meta, sizeof(uint16_t) * p->n, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < p->n; r++)
      if (meta[r] == kMetaGeneric) return MPB_OK;
  }
  std::vector<int> pat(static_cast<size_t>(p->npat) * kPatStride);
  MPB_CUDA(cudaMemcpy(pat.data(), p->d_pat, sizeof(int) * pat.size(), cudaMemcpyDeviceToHost));
  std::vector<int> offs;
  for (int q = 0; q < p->npat; q++) {
    const int *P = &pat[static_cast<size_t>(q) * kPatStride];
    for (int u = 0; u < (P[0] & 0xFF); u++) offs.push_back(P[1 + u]);
  }
  std::sort(offs.begin(), offs.end());
  offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
  if (static_cast<int>(offs.size()) != kDiaSlots || offs[kDiaDiag] != 0) return MPB_OK;
  std::vector<signed char> pslot(static_cast<size_t>(p->npat) * kSlots, 0);
  for (int q = 0; q < p->npat; q++) {
    const int *P = &pat[static_cast<size_t>(q) * kPatStride];
    const int len = P[0] & 0xFF;
    if (len > kDiaSlots) return MPB_OK;
    for (int u = 0; u < len; u++) {
      const int j = static_cast<int>(std::lower_bound(offs.begin(), offs.end(), P[1 + u]) - offs.begin());
      if (u > 0 && P[1 + u] <= P[u]) return MPB_OK;  // (stored order must ascend)
      pslot[static_cast<size_t>(q) * kSlots + u] = static_cast<signed char>(j);
    }
  }
  cudaFree(p->d_dmeta);
  cudaFree(p->d_pslot);
  p->d_dmeta = nullptr;
  p->d_pslot = nullptr;
  unsigned int *d_any = nullptr;
  MPB_CUDA(cudaMalloc(&p->d_dmeta, sizeof(uint16_t) * p->n));
  MPB_CUDA(cudaMalloc(&p->d_pslot, pslot.size()));
  MPB_CUDA(cudaMalloc(&d_any, sizeof(unsigned int)));
  MPB_CUDA(cudaMemcpy(p->d_pslot, pslot.data(), pslot.size(), cudaMemcpyHostToDevice));
  MPB_CUDA(cudaMemsetAsync(d_any, 0, sizeof(unsigned int), h->user));
  k_dia_meta<<<elt_blocks(p->n), kEltThreads, 0, h->user>>>(p->n, p->d_meta, p->d_pat, p->d_pslot, p->d_dmeta, d_any);
  MPB_LAUNCHED(h);
  unsigned int any = 0;
  MPB_CUDA(cudaMemcpyAsync(&any, d_any, sizeof(any), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  cudaFree(d_any);
  for (int k = 0; k < kDiaSlots; k++) p->dia_off[k] = offs[k];
  p->dia_ibany = static_cast<int>(any);
  p->dia_at = (p->ib_nnz + 63) & ~int64_t(63);  // (256-byte aligned for either precision)
  p->dia_entries = ((p->n + 31) / 32) * 32 * kDiaSlots;  // (whole 32-row slices)
  constexpr unsigned int kNear = (1u << (kDiaDiag - 1)) | (1u << kDiaDiag) | (1u << (kDiaDiag + 1));
  p->near_at = p->dia_at + p->dia_entries;      // (a multiple of 64 entries again)
  p->near_entries = (!p->large && (any & ~kNear) == 0u) ? p->n * kNearSlots : 0;
  p->dia_layout = true;
  p->dia_ok = !p->large;
  p->dia_big = p->large != 0;
  return MPB_OK;
}

int mpb_plan_bind_sell(mpb_handle *h, mpb_plan *p, const mpb_sell *sell) {
  if (!h || !p || !sell || sell->n != p->n) return MPB_ERR_ARG;
  if (p->bound == sell && p->d_meta) return MPB_OK;
  MPB_CUDA(cudaSetDevice(h->device));
  if (!p->d_meta) MPB_CUDA(cudaMalloc(&p->d_meta, sizeof(uint16_t) * p->n));
  k_build_meta<<<elt_blocks(p->n), kEltThreads, 0, h->user>>>(p->n, sell->d_pid, sell->d_pat, p->d_boff,
                                                            static_cast<int>(p->nb), p->d_meta);
  MPB_LAUNCHED(h);
  p->d_pat = sell->d_pat;
  p->npat = sell->npat;
  p->ks = sell->max_len <= 7 ? 7 : kSlots;
  if (!p->large) {
    k_tile_generic<<<static_cast<unsigned>(p->ntiles), kTileRows, 0, h->user>>>(p->d_td, p->d_meta);
    MPB_LAUNCHED(h);
  }
  // in-block SELL layout: per-row in-block counts -> slice widths -> pack
  const int64_t n = p->n, ns = (n + 31) / 32;
  int *d_cnt = nullptr;
  MPB_CUDA(cudaMalloc(&d_cnt, sizeof(int) * n));
  k_ib_count<<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, sell->d_sp, sell->d_col, p->d_boff,
                                                       static_cast<int>(p->nb), d_cnt);
  MPB_LAUNCHED(h);
  std::vector<int> cnt(n);
  MPB_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int) * n, cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  cudaFree(d_cnt);
  p->max_ib_row = 0;
  for (int64_t r = 0; r < n; r++) p->max_ib_row = std::max(p->max_ib_row, cnt[r]);
  std::vector<int> ib_sp(ns + 1);
  int64_t acc = 0;
  for (int64_t sl = 0; sl < ns; sl++) {
    int wdt = 0;
    for (int64_t r = 32 * sl; r < std::min<int64_t>(n, 32 * sl + 32); r++) wdt = std::max(wdt, cnt[r]);
    ib_sp[sl] = static_cast<int>(acc);
    acc += 32 * wdt;
    if (acc >= (int64_t(1) << 31)) return MPB_ERR_INDEX32;
  }
  ib_sp[ns] = static_cast<int>(acc);
  cudaFree(p->d_ib_sp);
  cudaFree(p->d_ib_col);
  p->d_ib_sp = nullptr;
  p->d_ib_col = nullptr;
  MPB_CUDA(cudaMalloc(&p->d_ib_sp, sizeof(int) * (ns + 1)));
  MPB_CUDA(cudaMalloc(&p->d_ib_col, sizeof(int) * std::max<int64_t>(acc, 1)));
  MPB_CUDA(cudaMemcpy(p->d_ib_sp, ib_sp.data(), sizeof(int) * (ns + 1), cudaMemcpyHostToDevice));
  MPB_CUDA(cudaMemsetAsync(p->d_ib_col, 0xff, sizeof(int) * std::max<int64_t>(acc, 1), h->user));
  k_ib_pack<int><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, sell->d_sp, sell->d_col, p->d_boff,
                                                           static_cast<int>(p->nb), p->d_ib_sp, sell->d_col,
                                                           p->d_ib_col);
  MPB_LAUNCHED(h);
  p->ib_nnz = acc;
  // tile descriptors gain their in-block entry ranges
  std::vector<TileDesc> td(p->ntiles);
  MPB_CUDA(cudaStreamSynchronize(h->user));
  MPB_CUDA(cudaMemcpy(td.data(), p->d_td, sizeof(TileDesc) * p->ntiles, cudaMemcpyDeviceToHost));
  int mx = 0;
  p->ngeneric = 0;
  for (auto &d : td) {
    d.ie0 = ib_sp[d.s0];
    d.ie1 = ib_sp[d.s1];
    mx = std::max(mx, d.ie1 - d.ie0);
    p->ngeneric += d.ngen;
  }
  p->max_tile_ib = mx;
  MPB_CUDA(cudaMemcpy(p->d_td, td.data(), sizeof(TileDesc) * p->ntiles, cudaMemcpyHostToDevice));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  p->bound = sell;
  // Symmetric offset-slot SpMV: the offsets must be a symmetric set with at
  // most kSymMax nonnegative members (the values are checked per operator)
  p->sym_S = 0;
  p->sym_key = nullptr;
  p->sym_ok = false;
  // off by default (MPB_SYM=1): on C2 it moves 50 MB less per SpMV (ncu:
  // 97 MB against 147 MB) but runs 41 us against 32.7 us for the SELL kernel
  // (profiles/r02_notes.md)
  static const bool no_sym = !(std::getenv("MPB_SYM") && std::atoi(std::getenv("MPB_SYM")) != 0);
  if (!no_sym && !p->large && p->ngeneric == 0 && p->npat > 0) {
    std::vector<int> pat(static_cast<size_t>(p->npat) * kPatStride);
    MPB_CUDA(cudaMemcpy(pat.data(), p->d_pat, sizeof(int) * pat.size(), cudaMemcpyDeviceToHost));
    std::vector<int> offs;
    for (int q = 0; q < p->npat; q++) {
      const int *P = &pat[static_cast<size_t>(q) * kPatStride];
      for (int u = 0; u < (P[0] & 0xFF); u++) offs.push_back(P[1 + u]);
    }
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    bool symset = !offs.empty();
    for (int o : offs) symset = symset && std::binary_search(offs.begin(), offs.end(), -o);
    std::vector<int> pos;
    for (int o : offs)
      if (o >= 0) pos.push_back(o);
    if (symset && !pos.empty() && pos[0] == 0 && (static_cast<int>(pos.size()) == 4 || static_cast<int>(pos.size()) == 6)) {
      const int S = static_cast<int>(pos.size());
      std::vector<uint16_t> mask(p->npat, 0);
      for (int q = 0; q < p->npat; q++) {
        const int *P = &pat[static_cast<size_t>(q) * kPatStride];
        for (int u = 0; u < (P[0] & 0xFF); u++) {
          const int j = static_cast<int>(std::lower_bound(offs.begin(), offs.end(), P[1 + u]) - offs.begin());
          mask[q] |= static_cast<uint16_t>(1u << j);
        }
      }
      cudaFree(p->d_pmask);
      p->d_pmask = nullptr;
      MPB_CUDA(cudaMalloc(&p->d_pmask, sizeof(uint16_t) * p->npat));
      MPB_CUDA(cudaMemcpy(p->d_pmask, mask.data(), sizeof(uint16_t) * p->npat, cudaMemcpyHostToDevice));
      p->sym_S = S;
      for (int k = 0; k < S; k++) p->sym_d[k] = pos[k];
    }
  }
  // Gather windows: the distinct column offsets of the row patterns,
  // clustered into <= kMaxWin row intervals [a, b] (a new window where the
  // gap to the previous offset exceeds a tile); a pass after the first then
  // stages z_in rows [lo + a, hi + b) of every window with TMA and gathers
  // from shared memory.  Needs pattern rows only and tiles starting at a
  // multiple of 4 rows (16-byte aligned fp32 / fp64 windows at a fixed skew).
  p->win = WinSet{};
  bool aligned = true;
  for (auto &d : td) aligned = aligned && (d.lo % 4 == 0);
  // off by default (MPB_WIN=1): the larger stages made the last pass slower
  // on C2 (39.2 us against 37.1 without, 37.2 against 33.0 with the full-tile
  // path; profiles/r02_notes.md)
  static const bool no_win = !(std::getenv("MPB_WIN") && std::atoi(std::getenv("MPB_WIN")) != 0);
  if (!p->large && p->ngeneric == 0 && aligned && p->npat > 0 && !no_win) {
    std::vector<int> pat(static_cast<size_t>(p->npat) * kPatStride);
    MPB_CUDA(cudaMemcpy(pat.data(), p->d_pat, sizeof(int) * pat.size(), cudaMemcpyDeviceToHost));
    std::vector<int> offs;
    for (int q = 0; q < p->npat; q++) {
      const int *P = &pat[static_cast<size_t>(q) * kPatStride];
      for (int u = 0; u < (P[0] & 0xFF); u++) offs.push_back(P[1 + u]);
    }
    offs.push_back(0);
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    WinSet w{};
    int rows = 0;
    bool ok = true;
    for (int o : offs) {
      if (w.n > 0 && o - w.b[w.n - 1] <= kTileRows) {
        w.b[w.n - 1] = o;
        continue;
      }
      if (w.n == kMaxWin) {
        ok = false;
        break;
      }
      w.a[w.n] = w.b[w.n] = o;
      w.n++;
    }
    for (int k = 0; k < w.n; k++) rows += kTileRows + w.b[k] - w.a[k];
    if (ok && rows <= kWinMaxRows) p->win = w;
    if (std::getenv("MPB_VERBOSE")) {
      std::fprintf(stderr, "[mpb] gather windows (off by default):");
      for (int k = 0; k < w.n; k++) std::fprintf(stderr, " [%d, %d]", w.a[k], w.b[k]);
      std::fprintf(stderr, " (%d rows)%s\n", rows, p->win.n ? "" : " -- not used");
    }
  }
  {
    const int rc = plan_dia(h, p);
    if (rc) return rc;
  }
  return plan_wave(h, p, td);
}

// entries of the plan-packed value buffer: the in-block SELL values, then
// (stencil plans, dia_ok) the offset-slot values at entry dia_at
int64_t mpb_plan_inblock_nnz(const mpb_plan *p) {
  if (!p || !p->bound) return MPB_ERR_LAYOUT;
  return p->dia_layout ? p->near_at + p->near_entries : p->ib_nnz;
}

template <typename T>
static int pack_ib_impl(mpb_handle *h, const mpb_plan *p, const T *sell_val, T *ib_val) {
  if (!h || !p || !sell_val || !ib_val) return MPB_ERR_ARG;
  if (!p->bound || !p->d_ib_sp) return MPB_ERR_LAYOUT;
  MPB_CUDA(cudaMemsetAsync(ib_val, 0, sizeof(T) * std::max<int64_t>(p->ib_nnz, 1), h->user));
  k_ib_pack<T><<<elt_blocks(p->n), kEltThreads, 0, h->user>>>(p->n, p->bound->d_sp, p->bound->d_col, p->d_boff,
                                                             static_cast<int>(p->nb), p->d_ib_sp, sell_val, ib_val);
  MPB_LAUNCHED(h);
  if (p->dia_layout) {  // the offset-slot values follow at entry dia_at
    MPB_CUDA(cudaMemsetAsync(ib_val + p->ib_nnz, 0, sizeof(T) * (p->dia_at + p->dia_entries - p->ib_nnz), h->user));
    k_dia_pack<T><<<elt_blocks(p->n), kEltThreads, 0, h->user>>>(p->n, p->bound->d_sp, sell_val, p->d_meta, p->d_pat,
                                                                p->d_pslot, ib_val + p->dia_at);
    MPB_LAUNCHED(h);
    if (p->near_entries > 0) {
      k_dia_near<T><<<elt_blocks(p->n), kEltThreads, 0, h->user>>>(p->n, ib_val + p->dia_at, ib_val + p->near_at);
      MPB_LAUNCHED(h);
    }
  }
  return MPB_OK;
}

int mpb_plan_pack_inblock_f64(mpb_handle *h, const mpb_plan *p, const double *sell_val, double *ib_val) {
  return pack_ib_impl<double>(h, p, sell_val, ib_val);
}

int mpb_plan_pack_inblock_f32(mpb_handle *h, const mpb_plan *p, const float *sell_val, float *ib_val) {
  return pack_ib_impl<float>(h, p, sell_val, ib_val);
}

int mpb_plan_info(const mpb_plan *p, int64_t *h_ntiles, int *h_large, int64_t *h_max_tile_nnz) {
  if (!p) return MPB_ERR_ARG;
  if (h_ntiles) *h_ntiles = p->ntiles;
  if (h_large) *h_large = p->large;
  if (h_max_tile_nnz) *h_max_tile_nnz = p->max_tile_nnz;
  return MPB_OK;
}

// ---- GPU-side problem assembly -------------------------------------------
int64_t mpb_stencil_nnz(int64_t n) { return n < 2 ? (n == 1 ? 1 : 0) : stencil_row_ptr(n * n * n, n); }

int mpb_assemble_stencil(mpb_handle *h, int64_t n, const double *kappa, double wx, double wy, double wz,
                         double scale, int32_t *row_ptr, int32_t *col_idx, double *values) {
  if (!h || n < 2 || !kappa || !row_ptr || !col_idx || !values) return MPB_ERR_ARG;
  if (n * n * n >= (int64_t(1) << 31) - 1 || mpb_stencil_nnz(n) >= (int64_t(1) << 31)) return MPB_ERR_INDEX32;
  MPB_CUDA(cudaSetDevice(h->device));
  k_stencil<<<elt_blocks(n * n * n), kEltThreads, 0, h->user>>>(n, kappa, wx, wy, wz, scale, row_ptr, col_idx,
                                                                 values);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int mpb_expand_3t(mpb_handle *h, int64_t ncell, const int32_t *rp1, const int32_t *col1, const double *val1,
                  const double *w_re, const double *w_ei, double time_term, int32_t *row_ptr, int32_t *col_idx,
                  double *values) {
  if (!h || ncell < 1 || !rp1 || !col1 || !val1 || !w_re || !w_ei || !row_ptr || !col_idx || !values)
    return MPB_ERR_ARG;
  if (3 * ncell >= (int64_t(1) << 31) - 1) return MPB_ERR_INDEX32;
  MPB_CUDA(cudaSetDevice(h->device));
  k_expand_3t<<<elt_blocks(ncell), kEltThreads, 0, h->user>>>(ncell, rp1, col1, val1, w_re, w_ei, time_term, row_ptr,
                                                              col_idx, values);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int mpb_splitmix64_uniform(mpb_handle *h, uint64_t seed, int64_t count, double a, double b, double *out) {
  if (!h || count < 0 || (count > 0 && !out)) return MPB_ERR_ARG;
  if (count == 0) return MPB_OK;
  MPB_CUDA(cudaSetDevice(h->device));
  k_splitmix64<<<elt_blocks(count), kEltThreads, 0, h->user>>>(seed, count, a, b, out);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int mpb_plan_layout_info(const mpb_plan *p, int *h_npat, int64_t *h_ngeneric) {
  if (!p || !p->bound) return MPB_ERR_ARG;
  if (h_npat) *h_npat = p->npat;
  if (h_ngeneric) *h_ngeneric = p->ngeneric;
  return MPB_OK;
}

int mpb_plan_offset_slot_info(const mpb_plan *p, int *h_slots, int *h_inblock_slots, int *h_near) {
  if (!p || !p->bound) return MPB_ERR_ARG;
  if (h_slots) *h_slots = p->dia_layout ? kDiaSlots : 0;
  if (h_inblock_slots) *h_inblock_slots = p->dia_layout ? p->dia_ibany : 0;
  if (h_near) *h_near = (p->dia_ok && p->near_entries > 0) ? 1 : 0;
  return MPB_OK;
}

// ---- backend kernels -------------------------------------------------------
int mpb_csr_matvec_f64(mpb_handle *h, int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const double *val,
                       const double *x, double *y) {
  if (!h || n < 0 || (n > 0 && (!row_ptr || !y))) return MPB_ERR_ARG;
  if (n == 0) return MPB_OK;
  k_matvec<double><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, row_ptr, col_idx, val, x, y);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int mpb_csr_matvec_f32(mpb_handle *h, int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const float *val,
                       const float *x, float *y) {
  if (!h || n < 0 || (n > 0 && (!row_ptr || !y))) return MPB_ERR_ARG;
  if (n == 0) return MPB_OK;
  k_matvec<float><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, row_ptr, col_idx, val, x, y);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

template <typename T>
static int sweeps_impl(mpb_handle *h, const int32_t *rp, const int32_t *ci, const T *val, const uint8_t *mask,
                       const T *diag, int t, const T *r, T *y, T *tmp, int64_t rs, int64_t re) {
  if (!h || !rp || !diag || !r || !y || !tmp || rs < 0 || re < rs) return MPB_ERR_ARG;
  if (re == rs) return MPB_OK;
  const int g = elt_blocks(re - rs);
  k_msweep_init<T><<<g, kEltThreads, 0, h->user>>>(rs, re, r, diag, y);
  MPB_LAUNCHED(h);
  for (int s = 0; s < t - 1; s++) {
    k_msweep_tmp<T><<<g, kEltThreads, 0, h->user>>>(rs, re, rp, ci, val, mask, y, tmp);
    MPB_LAUNCHED(h);
    k_msweep_upd<T><<<g, kEltThreads, 0, h->user>>>(rs, re, r, diag, tmp, y);
    MPB_LAUNCHED(h);
  }
  return MPB_OK;
}

int mpb_block_jacobi_sweeps_f64(mpb_handle *h, const int32_t *row_ptr, const int32_t *col_idx, const double *val,
                                const uint8_t *in_block, const double *diag, int t, const double *r, double *y,
                                double *tmp, int64_t row_start, int64_t row_end) {
  return sweeps_impl<double>(h, row_ptr, col_idx, val, in_block, diag, t, r, y, tmp, row_start, row_end);
}

int mpb_block_jacobi_sweeps_f32(mpb_handle *h, const int32_t *row_ptr, const int32_t *col_idx, const float *val,
                                const uint8_t *in_block, const float *diag, int t, const float *r, float *y,
                                float *tmp, int64_t row_start, int64_t row_end) {
  return sweeps_impl<float>(h, row_ptr, col_idx, val, in_block, diag, t, r, y, tmp, row_start, row_end);
}

// Global sum of nt tile partials in the order of include/mpbjac_order.h:
// one level, or chunk sums into csum (nt/256 + 1 entries of scratch) and
// the final level over them, into *out.
template <typename ACC>
static int launch_fin(mpb_handle *h, const ACC *part, int64_t nt, ACC *csum, ACC *out) {
  if (!two_level(nt)) {
    k_fin<ACC><<<1, kFinThreads, 0, h->user>>>(part, nt, out);
    MPB_LAUNCHED(h);
    return MPB_OK;
  }
  const int64_t nch = (nt + kChunkTiles - 1) / kChunkTiles;
  const int per = kTileThreads / 32;
  k_chunk_sums<ACC><<<static_cast<unsigned>((nch + per - 1) / per), kTileThreads, 0, h->user>>>(part, nt, csum);
  MPB_LAUNCHED(h);
  k_fin<ACC><<<1, kFinThreads, 0, h->user>>>(csum, nch, out);
  MPB_LAUNCHED(h);
  return MPB_OK;
}
static size_t chunk_scratch(size_t es, int64_t nt) { return al256(es * ((nt + kChunkTiles - 1) / kChunkTiles + 1)); }

template <typename T, typename ACC, bool SQ>
static int tile_reduce(mpb_handle *h, const mpb_plan *plan, int64_t n, const T *x, const T *y, ACC *h_out) {
  if (!h || !h_out || n < 0) return MPB_ERR_ARG;
  if (n == 0) {
    *h_out = ACC(0);
    return MPB_OK;
  }
  if (plan && plan->n != n) return MPB_ERR_SHAPE;
  const int64_t nt = plan ? plan->ntiles : (n + kTileRows - 1) / kTileRows;
  int rc = ensure_scratch(h, al256(sizeof(ACC) * (nt + 1)) + chunk_scratch(sizeof(ACC), nt) + 256);
  if (rc) return rc;
  ACC *part = static_cast<ACC *>(h->scratch);
  ACC *csum = reinterpret_cast<ACC *>(static_cast<char *>(h->scratch) + al256(sizeof(ACC) * (nt + 1)));
  ACC *res = reinterpret_cast<ACC *>(reinterpret_cast<char *>(csum) + chunk_scratch(sizeof(ACC), nt));
  k_tile_dot<T, ACC, SQ><<<static_cast<unsigned>(nt), kTileThreads, 0, h->user>>>(n, plan ? plan->d_tile_lo : nullptr,
                                                                                 x, y, part);
  MPB_LAUNCHED(h);
  if ((rc = launch_fin<ACC>(h, part, nt, csum, res))) return rc;
  MPB_CUDA(cudaMemcpyAsync(h_out, res, sizeof(ACC), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  return MPB_OK;
}

int mpb_dot_f64(mpb_handle *h, const mpb_plan *plan, int64_t n, const double *x, const double *y, double *h_out) {
  return tile_reduce<double, double, false>(h, plan, n, x, y, h_out);
}
int mpb_dot_f32(mpb_handle *h, const mpb_plan *plan, int64_t n, const float *x, const float *y, float *h_out) {
  return tile_reduce<float, float, false>(h, plan, n, x, y, h_out);
}
int mpb_norm_sq_f64(mpb_handle *h, const mpb_plan *plan, int64_t n, const double *x, double *h_out) {
  return tile_reduce<double, double, true>(h, plan, n, x, x, h_out);
}
int mpb_norm_sq_f32(mpb_handle *h, const mpb_plan *plan, int64_t n, const float *x, double *h_out) {
  return tile_reduce<float, double, true>(h, plan, n, x, x, h_out);
}

// ---- conversions / setup -----------------------------------------------------
static int narrow_impl(mpb_handle *h, int64_t n, const double *src, float *dst, int64_t *h_cnt, int64_t *h_first) {
  if (!h || n < 0) return MPB_ERR_ARG;
  int rc = ensure_scratch(h, 256);
  if (rc) return rc;
  unsigned long long *cnt = static_cast<unsigned long long *>(h->scratch);
  long long *first = reinterpret_cast<long long *>(cnt + 1);
  const long long init[2] = {0, (long long)INT64_MAX};
  MPB_CUDA(cudaMemcpyAsync(cnt, init, sizeof(init), cudaMemcpyHostToDevice, h->user));
  if (n > 0) {
    k_narrow<<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, src, dst, cnt, first);
    MPB_LAUNCHED(h);
  }
  long long out[2];
  MPB_CUDA(cudaMemcpyAsync(out, cnt, sizeof(out), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  if (h_cnt) *h_cnt = out[0];
  if (h_first) *h_first = out[0] ? out[1] : -1;
  return MPB_OK;
}

int mpb_narrow_f64_f32(mpb_handle *h, int64_t n, const double *src, float *dst, int64_t *h_overflow_count,
                       int64_t *h_first_index) {
  return narrow_impl(h, n, src, dst, h_overflow_count, h_first_index);
}

int mpb_convert_values_f32(mpb_handle *h, int64_t nnz, const double *val64, float *val32, int64_t *h_overflow_count,
                           int64_t *h_first_index) {
  return narrow_impl(h, nnz, val64, val32, h_overflow_count, h_first_index);
}

int mpb_widen_f32_f64(mpb_handle *h, int64_t n, const float *src, double *dst) {
  if (!h || n < 0) return MPB_ERR_ARG;
  if (n == 0) return MPB_OK;
  k_widen<<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, src, dst);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

template <typename T>
static int diag_impl(mpb_handle *h, int64_t n, const int32_t *rp, const int32_t *ci, const T *val, T *diag,
                     int64_t *h_missing, int64_t *h_zero) {
  if (!h || n < 1 || !rp || !ci || !val || !diag) return MPB_ERR_ARG;
  int rc = ensure_scratch(h, 256);
  if (rc) return rc;
  long long *flags = static_cast<long long *>(h->scratch);
  const long long init[2] = {(long long)INT64_MAX, (long long)INT64_MAX};
  MPB_CUDA(cudaMemcpyAsync(flags, init, sizeof(init), cudaMemcpyHostToDevice, h->user));
  k_setup_diag<T><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, rp, ci, val, diag, flags, flags + 1);
  MPB_LAUNCHED(h);
  long long out[2];
  MPB_CUDA(cudaMemcpyAsync(out, flags, sizeof(out), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  if (h_missing) *h_missing = out[0] == (long long)INT64_MAX ? -1 : out[0];
  if (h_zero) *h_zero = out[1] == (long long)INT64_MAX ? -1 : out[1];
  return MPB_OK;
}

int mpb_setup_diag_f64(mpb_handle *h, int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const double *val64,
                       double *diag, int64_t *h_missing, int64_t *h_zero) {
  return diag_impl<double>(h, n, row_ptr, col_idx, val64, diag, h_missing, h_zero);
}

int mpb_setup_diag_f32(mpb_handle *h, int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const float *val32,
                       float *diag, int64_t *h_missing, int64_t *h_zero) {
  return diag_impl<float>(h, n, row_ptr, col_idx, val32, diag, h_missing, h_zero);
}


// ---- SELL-32 layout ------------------------------------------------------------
// Row-pattern dictionary of a SELL structure (see mpbjac_kernels.cuh): count
// the rows of every distinct (length, column offsets) pattern on the device,
// keep the kPatMax most frequent, then tag every row with its verified
// pattern id (or kPidGeneric).
static cudaError_t build_patterns(mpb_handle *h, mpb_sell *S) {
  const int64_t n = S->n;
  PatSlot *d_tab = nullptr;
  int *d_aux = nullptr;
  cudaError_t e = cudaMalloc(&d_tab, sizeof(PatSlot) * kPatHash);
  if (e == cudaSuccess) e = cudaMalloc(&d_aux, sizeof(int) * (kPatHash + kPatMax));
  if (e == cudaSuccess) e = cudaMalloc(&S->d_pat, sizeof(int) * kPatMax * kPatStride);
  if (e == cudaSuccess) e = cudaMalloc(&S->d_pid, std::max<int64_t>(n, 1));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_tab, 0, sizeof(PatSlot) * kPatHash, h->user);
  if (e == cudaSuccess) e = cudaMemsetAsync(S->d_pat, 0, sizeof(int) * kPatMax * kPatStride, h->user);
  if (e == cudaSuccess) {
    k_pat_insert<<<static_cast<unsigned>((n + 255) / 256), 256, 0, h->user>>>(n, S->d_sp, S->d_col, d_tab);
    h->launches++;
    e = cudaGetLastError();
  }
  std::vector<PatSlot> tab(kPatHash);
  if (e == cudaSuccess) e = cudaMemcpyAsync(tab.data(), d_tab, sizeof(PatSlot) * kPatHash, cudaMemcpyDeviceToHost,
                                            h->user);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->user);
  if (e == cudaSuccess) {
    std::vector<int> order;
    for (int i = 0; i < kPatHash; i++)
      if (tab[i].key != 0ull && tab[i].count > 0) order.push_back(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tab[a].count > tab[b].count; });
    if (order.size() > static_cast<size_t>(kPatMax)) order.resize(kPatMax);
    S->npat = static_cast<int>(order.size());
    std::vector<int> aux(kPatHash + kPatMax, -1);  // slot -> pid, then the representative rows
    for (int i = 0; i < S->npat; i++) {
      aux[order[i]] = i;
      aux[kPatHash + i] = tab[order[i]].rep;
    }
    e = cudaMemcpyAsync(d_aux, aux.data(), sizeof(int) * aux.size(), cudaMemcpyHostToDevice, h->user);
    if (e == cudaSuccess && S->npat > 0) {
      k_pat_fetch<<<1, kPatMax, 0, h->user>>>(d_aux + kPatHash, S->npat, S->d_sp, S->d_col, S->d_pat);
      h->launches++;
      e = cudaGetLastError();
    }
    S->max_len = 0;
    if (e == cudaSuccess && S->npat > 0) {
      std::vector<int> pat(static_cast<size_t>(S->npat) * kPatStride);
      e = cudaMemcpyAsync(pat.data(), S->d_pat, sizeof(int) * pat.size(), cudaMemcpyDeviceToHost, h->user);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->user);
      for (int i = 0; i < S->npat && e == cudaSuccess; i++)
        S->max_len = std::max(S->max_len, pat[static_cast<size_t>(i) * kPatStride] & 0xFF);
    }
    if (e == cudaSuccess) {
      k_pat_assign<<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, S->d_sp, S->d_col, d_tab, d_aux, S->d_pat,
                                                              S->d_pid);
      h->launches++;
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->user);
  }
  cudaFree(d_tab);
  cudaFree(d_aux);
  return e;
}

int mpb_sell_create(mpb_handle *h, int64_t n, const int64_t *h_row_ptr, const int32_t *row_ptr,
                    const int32_t *col_idx, mpb_sell **out) {
  if (!h || !out || !h_row_ptr || !row_ptr || !col_idx || n < 1) return MPB_ERR_ARG;
  *out = nullptr;
  if (n >= (int64_t(1) << 31) - 1) return MPB_ERR_INDEX32;
  const int64_t ns = (n + 31) / 32;
  std::vector<int> sp;
  if (!sell_slice_ptrs(n, h_row_ptr, sp)) return MPB_ERR_INDEX32;
  const int64_t acc = sp[ns];
  MPB_CUDA(cudaSetDevice(h->device));
  mpb_sell *S = new mpb_sell();
  S->n = n;
  S->nslices = ns;
  S->nnz = acc;
  cudaError_t e = cudaMalloc(&S->d_sp, sizeof(int) * (ns + 1));
  if (e == cudaSuccess) e = cudaMalloc(&S->d_col, sizeof(int) * std::max<int64_t>(acc, 1));
  if (e == cudaSuccess) e = cudaMemcpy(S->d_sp, sp.data(), sizeof(int) * (ns + 1), cudaMemcpyHostToDevice);
  // padding slots: column -1 (all bytes 0xff)
  if (e == cudaSuccess) e = cudaMemsetAsync(S->d_col, 0xff, sizeof(int) * std::max<int64_t>(acc, 1), h->user);
  if (e == cudaSuccess) {
    k_sell_pack<int><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, row_ptr, S->d_sp, col_idx, S->d_col);
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->user);
  if (e == cudaSuccess) e = build_patterns(h, S);
  if (e != cudaSuccess) {
    mpb_sell_destroy(S);
    return status_of(e);
  }
  *out = S;
  return MPB_OK;
}

int mpb_sell_destroy(mpb_sell *s) {
  if (!s) return MPB_OK;
  cudaFree(s->d_sp);
  cudaFree(s->d_col);
  cudaFree(s->d_pid);
  cudaFree(s->d_pat);
  delete s;
  return MPB_OK;
}

int64_t mpb_sell_nnz(const mpb_sell *s) { return s ? s->nnz : MPB_ERR_ARG; }

template <typename T>
static int sell_pack_impl(mpb_handle *h, const mpb_sell *S, const int32_t *rp, const T *csr, T *sell) {
  if (!h || !S || !rp || !csr || !sell) return MPB_ERR_ARG;
  MPB_CUDA(cudaMemsetAsync(sell, 0, sizeof(T) * std::max<int64_t>(S->nnz, 1), h->user));
  k_sell_pack<T><<<elt_blocks(S->n), kEltThreads, 0, h->user>>>(S->n, rp, S->d_sp, csr, sell);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int mpb_sell_pack_f64(mpb_handle *h, const mpb_sell *s, const int32_t *row_ptr, const double *csr_val,
                      double *sell_val) {
  return sell_pack_impl<double>(h, s, row_ptr, csr_val, sell_val);
}

int mpb_sell_pack_f32(mpb_handle *h, const mpb_sell *s, const int32_t *row_ptr, const float *csr_val,
                      float *sell_val) {
  return sell_pack_impl<float>(h, s, row_ptr, csr_val, sell_val);
}

// ---- preconditioner ----------------------------------------------------------
template <typename T>
static int apply_bufs_scratch(mpb_handle *h, const mpb_plan *p, int64_t n, size_t extra, ApplyBufs<T> &b,
                              char **extra_ptr) {
  const size_t v = al256(sizeof(T) * (n + 4));
  const size_t need = 2 * v + (p->large ? 4 * v : 0) + al256(extra);
  int rc = ensure_scratch(h, need);
  if (rc) return rc;
  char *base = static_cast<char *>(h->scratch);
  b.zA = (T *)base;
  b.zB = (T *)(base + v);
  size_t off = 2 * v;
  if (p->large) {
    b.res = (T *)(base + off);
    b.dg = (T *)(base + off + v);
    b.wA = (T *)(base + off + 2 * v);
    b.wB = (T *)(base + off + 3 * v);
    off += 4 * v;
  } else {
    b.res = b.dg = b.wA = b.wB = nullptr;
  }
  if (extra_ptr) *extra_ptr = base + off;
  return MPB_OK;
}

template <typename T>
static int apply_impl(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, int k, int t, const T *r, T *z) {
  int rc = check_sell(A, sizeof(T) == 8, sizeof(T) == 4);
  if (rc == MPB_OK) rc = check_bound(plan, A);
  if (rc) return rc;
  if (!h || !plan || !r || !z) return MPB_ERR_ARG;
  if (plan->n != A->n) return MPB_ERR_PARTITION;
  if (k < 1 || t < 1) return MPB_ERR_SWEEPS;
  ApplyBufs<T> b;
  rc = apply_bufs_scratch<T>(h, plan, A->n, 0, b, nullptr);
  if (rc) return rc;
  return launch_apply<T>(h, h->user, plan, A, k, t, nullptr, r, z, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                         b);
}

int mpb_bjac_apply_f64(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, int k, int t, const double *r,
                       double *z) {
  return apply_impl<double>(h, plan, A, k, t, r, z);
}

int mpb_bjac_apply_f32(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, int k, int t, const float *r,
                       float *z) {
  return apply_impl<float>(h, plan, A, k, t, r, z);
}

int mpb_fmp_apply(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, int k, int t, const double *r, double *z,
                  int64_t *h_overflow_count, int64_t *h_first_index) {
  int rc = check_sell(A, false, true);
  if (rc == MPB_OK) rc = check_bound(plan, A);
  if (rc) return rc;
  if (!h || !plan || !r || !z) return MPB_ERR_ARG;
  if (plan->n != A->n) return MPB_ERR_PARTITION;
  if (k < 1 || t < 1) return MPB_ERR_SWEEPS;
  ApplyBufs<float> b;
  char *extra;
  rc = apply_bufs_scratch<float>(h, plan, A->n, 256, b, &extra);
  if (rc) return rc;
  unsigned long long *cnt = reinterpret_cast<unsigned long long *>(extra);
  long long *first = reinterpret_cast<long long *>(extra + 8);
  const long long init[2] = {0, (long long)INT64_MAX};
  MPB_CUDA(cudaMemcpyAsync(cnt, init, sizeof(init), cudaMemcpyHostToDevice, h->user));
  rc = launch_apply<float>(h, h->user, plan, A, k, t, r, nullptr, nullptr, z, nullptr, cnt, first, nullptr, 0, b);
  if (rc) return rc;
  long long out[2];
  MPB_CUDA(cudaMemcpyAsync(out, cnt, sizeof(out), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  if (h_overflow_count) *h_overflow_count = out[0];
  if (h_first_index) *h_first_index = out[0] ? out[1] : -1;
  return MPB_OK;
}

template <typename T>
static int inner_impl(mpb_handle *h, const mpb_csr *A, const T *val, int64_t lo, int64_t hi, int t, const T *rb,
                      T *yb) {
  int rc = check_csr(A);
  if (rc) return rc;
  if (!h || !val || !rb || !yb || lo < 0 || hi > A->n || hi <= lo) return MPB_ERR_ARG;
  if (t < 1) return MPB_ERR_SWEEPS;
  const int64_t m = hi - lo;
  const size_t v = al256(sizeof(T) * (m + 4));
  rc = ensure_scratch(h, 2 * v);
  if (rc) return rc;
  T *db = static_cast<T *>(h->scratch);
  T *tmp = reinterpret_cast<T *>(static_cast<char *>(h->scratch) + v);
  const int g = elt_blocks(m);
  k_inner_init<T><<<g, kEltThreads, 0, h->user>>>((int)lo, (int)hi, A->row_ptr, A->col_idx, val, rb, db, yb);
  MPB_LAUNCHED(h);
  for (int s = 1; s < t; s++) {
    k_inner_sweep<T><<<g, kEltThreads, 0, h->user>>>((int)lo, (int)hi, A->row_ptr, A->col_idx, val, rb, db, yb, tmp);
    MPB_LAUNCHED(h);
    MPB_CUDA(cudaMemcpyAsync(yb, tmp, sizeof(T) * m, cudaMemcpyDeviceToDevice, h->user));
  }
  return MPB_OK;
}

int mpb_bjac_inner_apply_f64(mpb_handle *h, const mpb_csr *A, int64_t row_lo, int64_t row_hi, int t,
                             const double *r_b, double *y_b) {
  return inner_impl<double>(h, A, A ? A->val64 : nullptr, row_lo, row_hi, t, r_b, y_b);
}

int mpb_bjac_inner_apply_f32(mpb_handle *h, const mpb_csr *A, int64_t row_lo, int64_t row_hi, int t,
                             const float *r_b, float *y_b) {
  return inner_impl<float>(h, A, A ? A->val32 : nullptr, row_lo, row_hi, t, r_b, y_b);
}

// ---- the PCG loop ------------------------------------------------------------
int64_t mpb_solve_workspace_bytes(const mpb_plan *plan, int64_t n) {
  if (!plan || n != plan->n) return MPB_ERR_ARG;
  return static_cast<int64_t>(carve(plan, n, nullptr).bytes);
}

// KS = 7 (7-point stencils) with or without generic rows; KS = 9 (e.g. 3-T) always with
static void (*spmv_kernel(const mpb_plan *p))(SpmvArgs) {
  if (two_level(p->ntiles)) {
    if (p->ks == 7) return p->ngeneric > 0 ? k_spmv_pq<7, true, true> : k_spmv_pq<7, false, true>;
    return k_spmv_pq<kSlots, true, true>;
  }
  if (p->ks == 7) return p->ngeneric > 0 ? k_spmv_pq<7, true> : k_spmv_pq<7, false>;
  return k_spmv_pq<kSlots, true>;
}

static TileGeom spmv_geom(const mpb_plan *p) {
  TileGeom g = geom_for<double>(p);
  g.ns = pick_stages(spmv_kernel(p), spmv_layout(g).bytes);
  return g;
}

static uint32_t spmv_dyn_smem(const mpb_plan *p) {
  const TileGeom g = spmv_geom(p);
  return g.ns * spmv_layout(g).bytes;
}

// The symmetric offset-slot layout of the operator's values (k_spmv_sym):
// built once per operator value array when the plan's offsets allow it and
// the values are symmetric bit for bit (one-GPU solves only: a slab's ghost
// rows are not row + offset).  Returns whether it is usable.
static bool ensure_sym(mpb_handle *h, mpb_plan *p, const mpb_csr *A, cudaStream_t s) {
  if (p->sym_S == 0) return false;
  const double *vals = op_vals(A);
  if (p->sym_key == vals) return p->sym_ok;
  p->sym_key = vals;
  p->sym_ok = false;
  unsigned long long *d_bad = nullptr, bad = 1;
  if (cudaMalloc(&d_bad, sizeof(unsigned long long)) != cudaSuccess) return false;
  cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s);
  k_sym_check<<<elt_blocks(A->n), kEltThreads, 0, s>>>(A->n, A->sell->d_sp, vals, p->d_meta, p->d_pat, d_bad);
  cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFree(d_bad);
  if (cudaGetLastError() != cudaSuccess || bad != 0) return false;
  cudaFree(p->d_U);
  p->d_U = nullptr;
  if (cudaMalloc(&p->d_U, sizeof(double) * p->sym_S * A->n) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  SpmvArgs da{};
  for (int k = 0; k < p->sym_S; k++) da.d[k] = p->sym_d[k];
  k_sym_build<<<elt_blocks(A->n), kEltThreads, 0, s>>>(A->n, A->sell->d_sp, vals, p->d_meta, p->d_pat, p->sym_S, da,
                                                       p->d_U);
  h->launches += 2;
  p->sym_ok = cudaGetLastError() == cudaSuccess;
  return p->sym_ok;
}

static void (*spmv_sym_kernel(const mpb_plan *p))(SpmvArgs) {
  const bool two = two_level(p->ntiles);
  if (p->sym_S == 4) return two ? k_spmv_sym<4, true> : k_spmv_sym<4, false>;
  return two ? k_spmv_sym<6, true> : k_spmv_sym<6, false>;
}

// pnew != null: p rebuilt from z and pold inside the SpMV (fused mode)
static SpmvArgs spmv_args(const mpb_handle *h, const mpb_plan *p, const mpb_csr *A, const SolveWs &w,
                          const double *pold = nullptr, double *pnew = nullptr) {
  SpmvArgs sa{};
  sa.sp = A->sell->d_sp;
  sa.scol = A->sell->d_col;
  sa.sval = op_vals(A);
  sa.meta = p->d_meta;
  sa.pat = p->d_pat;
  sa.td = p->d_td;
  sa.ctr = claim_ctr(h, 2);
  sa.g = spmv_geom(p);
  sa.p = w.p;
  sa.z32 = w.z32;
  sa.z64 = w.z64;
  sa.pold = pold;
  sa.pnew = pnew;
  sa.q = w.q;
  sa.part = w.part;
  sa.st = w.st;
  sa.csum = w.csum;
  // offset-slot layout of the operator: its plan-packed values (the
  // preconditioner's fp64 buffer when the operator is the preconditioner's matrix)
  const double *op_packed = A->op_sell_val64 ? A->op_ib_val64 : A->ib_val64;
  if (p->dia_ok && op_packed != nullptr) {
    sa.dval = op_packed + p->dia_at;
    sa.dmeta = p->d_dmeta;
    for (int u = 0; u < kDiaSlots; u++) sa.doff[u] = p->dia_off[u];
    if (red_mode(p)) {  // streamed one-level sum
      sa.part = red_part(p, p->n, sa.part);
      sa.g.red = 1;
    }
    auto kern = two_level(p->ntiles) ? k_spmv_dia<true> : k_spmv_dia<false>;
    sa.g.ns = pick_stages(kern, kDiaSpmvStage);
  }
  if (p->sym_ok && p->sym_key == op_vals(A) && p->d_U != nullptr) {
    sa.U = p->d_U;
    sa.pmask = p->d_pmask;
    sa.n = static_cast<int>(A->n);
    sa.S = p->sym_S;
    for (int k = 0; k < p->sym_S; k++) sa.d[k] = p->sym_d[k];
    sa.g.ns = pick_stages(spmv_sym_kernel(p), spmv_sym_layout(p->sym_S, p->sym_d).bytes);
  }
  return sa;
}

// the SpMV of an iteration: the symmetric offset-slot kernel when spmv_args
// bound a U layout, else the SELL kernel
static int launch_spmv(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const SpmvArgs &sa, bool pdl) {
  if (sa.dval != nullptr && sa.U == nullptr) {
    auto kern = two_level(p->ntiles) ? k_spmv_dia<true> : k_spmv_dia<false>;
    const uint32_t dyn = sa.g.ns * kDiaSpmvStage;
    MPB_CUDA(launch_k(pdl, kern, persistent_grid(kern, dyn, p->ntiles, kWsThreads), kWsThreads, dyn, s, sa));
  } else if (sa.U != nullptr) {
    auto kern = spmv_sym_kernel(p);
    const uint32_t dyn = sa.g.ns * spmv_sym_layout(sa.S, sa.d).bytes;
    MPB_CUDA(launch_k(pdl, kern, persistent_grid(kern, dyn, p->ntiles, kWsThreads), kWsThreads, dyn, s, sa));
  } else {
    const uint32_t dyn = spmv_dyn_smem(p);
    MPB_CUDA(launch_k(pdl, spmv_kernel(p), persistent_grid(spmv_kernel(p), dyn, p->ntiles, kWsThreads), kWsThreads,
                      dyn, s, sa));
  }
  MPB_LAUNCHED(h);
  return MPB_OK;
}

// One PCG iteration (solver.py:140-177): preconditioner of the branch(es)
// the policy can take (each gated on st->branch) with the fused rho step;
// p-update; SpMV with the pq step; x/r update with the relres / branch /
// convergence step; optional strided true residual.  Multi-GPU: halo
// exchanges before every gathering kernel, all-reduced scalar steps.
// Fused mode (single GPU, k >= 2, tile plan): the x/r update of iteration i
// and the first BJAC pass of iteration i+1 are one kernel (k_update_first).
// Multi-GPU: the fused iteration exchanges three halos (z after the last
// pass and p after the SpMV -- both gathered by the SpMV's p rebuild -- and
// z1 after the fused update), the unfused one two (z1, p).
static bool fused_mode(const mpb_plan *p, const mpb_solve_options *o, const DistCtx *) {
  static const bool off = std::getenv("MPB_NO_FUSE") != nullptr;
  return !off && o->k >= 2 && !p->large;
}
// wave mode (one GPU, fixed branch, k = 2): the iteration is the SpMV and
// the wave kernel (x/r update + first pass + the next last pass)
static bool wave_mode(const mpb_plan *p, const mpb_solve_options *o, const DistCtx *dc) {
  return dc == nullptr && fused_mode(p, o, dc) && o->k == 2 && p->wave_ok &&
         (o->kind == MPB_FIXED_LOW || o->kind == MPB_UNIFORM);
}

// Standalone first passes of the policy's branches (gated on st->branch and,
// z1_gate, on the fused update not having produced z1 already).
static int enqueue_first_passes(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const mpb_csr *A,
                                const mpb_solve_options *o, const SolveWs &w, const DistCtx *dc) {
  const bool high = o->kind != MPB_FIXED_LOW, low = o->kind != MPB_UNIFORM;
  int rc;
  if (high) {
    ApplyBufs<double> bb{w.zA64, w.zB64, w.res64, w.dg64, w.wA64, w.wB64};
    rc = launch_apply<double>(h, s, p, A, o->k, o->t, w.r, nullptr, w.z64, nullptr, w.part, nullptr, nullptr, w.st,
                              0, bb, dc, 0, 1, 1);  // (the z1 halo included: pass 0 is not the last)
    if (rc) return rc;
  }
  if (low) {
    ApplyBufs<float> bb{w.zA32, w.zB32, w.res32, w.dg32, w.wA32, w.wB32};
    rc = launch_apply<float>(h, s, p, A, o->k, o->t, w.r, nullptr, w.z32, nullptr, w.part, &w.st->ovf_count,
                             &w.st->ovf_first, w.st, 1, bb, dc, 0, 1, 1);
    if (rc) return rc;
  }
  return MPB_OK;
}

// it: iteration index inside the captured body (fused mode alternates the
// two p buffers; the body holds an even number of iterations)
static int enqueue_iteration(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const mpb_csr *A,
                             const mpb_solve_options *o, const SolveWs &w, const double *b, double *x,
                             const DistCtx *dc, int it) {
  const bool high = o->kind != MPB_FIXED_LOW, low = o->kind != MPB_UNIFORM;
  const unsigned nt = static_cast<unsigned>(p->ntiles);
  const bool fused = fused_mode(p, o, dc);
  // fixed-branch policies may stream their first tiles' matrix data before
  // the grid dependency wait (MPB_PREFETCH=1); measured 2 % slower on C2
  // (the early copies compete with the previous kernel's last tiles), so off
  static const bool use_pre = std::getenv("MPB_PREFETCH") != nullptr;
  const int pre = (fused && !(high && low) && use_pre) ? 1 : 0;
  int rc;
  // adaptive policies: the branch may have changed, invalidating the fused z1
  if (fused && high && low && (rc = enqueue_first_passes(h, s, p, A, o, w, dc))) return rc;
  const int from = fused ? 1 : 0;
  const bool wave = wave_mode(p, o, dc);  // the last pass ran in the previous wave kernel (or the prologue)
  if (high && !wave) {
    ApplyBufs<double> bb{w.zA64, w.zB64, w.res64, w.dg64, w.wA64, w.wB64};
    rc = launch_apply<double>(h, s, p, A, o->k, o->t, w.r, nullptr, w.z64, nullptr, w.part, nullptr, nullptr, w.st,
                              0, bb, dc, from, 1 << 30, 0, pre);
    if (rc) return rc;
  }
  if (low && !wave) {
    ApplyBufs<float> bb{w.zA32, w.zB32, w.res32, w.dg32, w.wA32, w.wB32};
    rc = launch_apply<float>(h, s, p, A, o->k, o->t, w.r, nullptr, w.z32, nullptr, w.part, &w.st->ovf_count,
                             &w.st->ovf_first, w.st, 1, bb, dc, from, 1 << 30, 0, pre);
    if (rc) return rc;
  }
  if (fused && dc) {  // the SpMV's p rebuild gathers z at ghost rows
    if (low && (rc = halo_exchange(dc, w.z32, 4, A->n, s))) return rc;
    if (high && (rc = halo_exchange(dc, w.z64, 8, A->n, s))) return rc;
  }
  if ((rc = dist_step(h, dc, w.st, kStepRho, 2, s))) return rc;
  const bool pdl = dc == nullptr;
  // fused mode: p = z + beta p_old is rebuilt inside the SpMV (no p-update
  // kernel); p ping-pongs between two buffers
  double *pcur = w.p;
  SpmvArgs sa;
  if (fused) {
    const double *pold = (it & 1) ? w.p2 : w.p;
    pcur = (it & 1) ? w.p : w.p2;
    sa = spmv_args(h, p, A, w, pold, pcur);
    sa.prefetch = pre;
    if (dc) sa.U = nullptr;  // (slabs: the ghost columns are not row + offset)
  } else {
    MPB_CUDA(launch_k(pdl, k_pupdate, persistent_grid(k_pupdate, 0, p->ntiles), kCtaThreads, 0, s,
                      static_cast<const TileDesc *>(p->d_td), static_cast<int>(nt), static_cast<const float *>(w.z32),
                      static_cast<const double *>(w.z64), w.p, static_cast<const SolverState *>(w.st)));
    MPB_LAUNCHED(h);
    if ((rc = halo_exchange(dc, w.p, 8, A->n, s))) return rc;
    sa = spmv_args(h, p, A, w);
    if (dc) sa.U = nullptr;
  }
  if ((rc = launch_spmv(h, s, p, sa, pdl))) return rc;
  if (fused && (rc = halo_exchange(dc, pcur, 8, A->n, s))) return rc;  // next iteration's p_old ghosts
  if ((rc = dist_step(h, dc, w.st, kStepPq, 2, s))) return rc;
  if (wave) {
    if (high && (rc = launch_wave<double>(h, s, p, A, o->t, w.zA64, w.z64, x, pcur, w.q, w.r, w.part, w.part2, w.gcnt,
                                          nullptr, nullptr, w.st, 0, pdl)))
      return rc;
    if (low && (rc = launch_wave<float>(h, s, p, A, o->t, w.zA32, w.z32, x, pcur, w.q, w.r, w.part, w.part2, w.gcnt,
                                        &w.st->ovf_count, &w.st->ovf_first, w.st, 1, pdl)))
      return rc;
  } else if (fused) {
    if (high && (rc = launch_update_first<double>(h, s, p, A, o->t, w.zA64, x, pcur, w.q, w.r, w.part, nullptr,
                                                  nullptr, w.st, 0, pre, pdl)))
      return rc;
    if (low && (rc = launch_update_first<float>(h, s, p, A, o->t, w.zA32, x, pcur, w.q, w.r, w.part,
                                                &w.st->ovf_count, &w.st->ovf_first, w.st, 1, pre, pdl)))
      return rc;
    if (dc) {  // z1 ghosts for the next last pass
      if (low && (rc = halo_exchange(dc, w.zA32, 4, A->n, s))) return rc;
      if (high && (rc = halo_exchange(dc, w.zA64, 8, A->n, s))) return rc;
    }
  } else {
    MPB_CUDA(launch_k(pdl, k_update, persistent_grid(k_update, 0, p->ntiles), kCtaThreads, 0, s,
                      static_cast<const TileDesc *>(p->d_td), static_cast<int>(nt), x,
                      static_cast<const double *>(w.p), static_cast<const double *>(w.q), w.r, w.part, w.st, w.csum, owners_poll(p->ntiles) ? 1 : 0));
    MPB_LAUNCHED(h);
  }
  if ((rc = dist_step(h, dc, w.st, fused ? kStepRrZ : kStepRr, 2, s))) return rc;
  if (o->true_stride > 0) {
    if ((rc = halo_exchange(dc, x, 8, A->n, s))) return rc;
    k_resid<true><<<persistent_grid(k_resid<true>, 0, p->ntiles), kCtaThreads, 0, s>>>(
        A->sell->d_sp, A->sell->d_col, op_vals(A), p->d_td, static_cast<int>(nt), b, x, nullptr, w.part, w.st, 1,
        kStepTrue, w.csum, owners_poll(p->ntiles) ? 1 : 0);
    MPB_LAUNCHED(h);
    if ((rc = dist_step(h, dc, w.st, kStepTrue, 1, s))) return rc;
  }
  return MPB_OK;
}

static int solve_impl(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                      const double *b, double *x, double *tr_relres, double *tr_true, int32_t *tr_branch,
                      double *tr_time, void *workspace, int64_t workspace_bytes, mpb_solve_result *res,
                      const DistCtx *dc);

int mpb_pcg_solve(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                  const double *b, double *x, double *tr_relres, double *tr_true, int32_t *tr_branch,
                  double *tr_time, void *workspace, int64_t workspace_bytes, mpb_solve_result *res) {
  return solve_impl(h, plan, A, opt, b, x, tr_relres, tr_true, tr_branch, tr_time, workspace, workspace_bytes, res,
                    nullptr);
}

int mpb_pcg_solve_dist(mpb_handle *h, const mpb_comm *comm, const mpb_halo *halo, const mpb_plan *plan,
                       const mpb_csr *A, const mpb_solve_options *opt, const double *b, double *x,
                       double *tr_relres, double *tr_true, int32_t *tr_branch, double *tr_time, void *workspace,
                       int64_t workspace_bytes, mpb_solve_result *res) {
  if (!comm || !halo) return MPB_ERR_ARG;
  if (halo->recv_lo < 0 || halo->recv_hi < 0 || halo->send_lo < 0 || halo->send_hi < 0) return MPB_ERR_ARG;
  if (halo->send_lo > A->n || halo->send_hi > A->n) return MPB_ERR_SHAPE;
  DistCtx dc{comm, *halo};
  const int rc = solve_impl(h, plan, A, opt, b, x, tr_relres, tr_true, tr_branch, tr_time, workspace,
                            workspace_bytes, res, &dc);
  if (rc != MPB_OK && comm->grp != nullptr) comm->grp->fail();  // release the other ranks
  return rc;
}

int64_t mpb_solve_workspace_bytes_dist(const mpb_plan *plan, int64_t n, int64_t ghosts) {
  if (!plan || n != plan->n || ghosts < 0) return MPB_ERR_ARG;
  return static_cast<int64_t>(carve(plan, n, nullptr, ghosts).bytes);
}

// ---- communicator ----------------------------------------------------------
int mpb_comm_unique_id(void *h_id) {
  if (!h_id) return MPB_ERR_ARG;
  NcclApi &N = nccl();
  if (!N.ok) return MPB_ERR_COMM;
  ncclUniqueId id;
  if (N.GetUniqueId(&id) != 0) return MPB_ERR_COMM;
  std::memcpy(h_id, &id, sizeof(id));
  return MPB_OK;
}

int mpb_comm_create(mpb_handle *h, int rank, int nranks, const void *h_id, mpb_comm **out) {
  if (!h || !h_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return MPB_ERR_ARG;
  *out = nullptr;
  NcclApi &N = nccl();
  if (!N.ok) return MPB_ERR_COMM;
  MPB_CUDA(cudaSetDevice(h->device));
  ncclUniqueId id;
  std::memcpy(&id, h_id, sizeof(id));
  mpb_comm *c = new mpb_comm();
  c->rank = rank;
  c->nranks = nranks;
  if (N.CommInitRank(&c->comm, nranks, id, rank) != 0) {
    delete c;
    return MPB_ERR_COMM;
  }
  *out = c;
  return MPB_OK;
}

int mpb_comm_destroy(mpb_comm *c) {
  if (!c) return MPB_OK;
  if (c->grp == nullptr) {
    NcclApi &N = nccl();
    if (N.ok && c->comm) N.CommDestroy(c->comm);
  }
  delete c;
  return MPB_OK;
}

int mpb_local_group_create(int device, int nranks, void **out) {
  if (!out || nranks < 1 || nranks > kMaxLocalRanks) return MPB_ERR_ARG;
  *out = nullptr;
  MPB_CUDA(cudaSetDevice(device));
  LocalGroup *g = new LocalGroup();
  g->nranks = nranks;
  g->slot.resize(nranks);
  cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete g;
    return status_of(e);
  }
  *out = g;
  return MPB_OK;
}

int mpb_local_group_destroy(void *group) {
  LocalGroup *g = static_cast<LocalGroup *>(group);
  if (!g) return MPB_OK;
  cudaStreamSynchronize(g->stream);
  cudaStreamDestroy(g->stream);
  delete g;
  cudaGetLastError();
  return MPB_OK;
}

void *mpb_local_group_stream(void *group) {
  LocalGroup *g = static_cast<LocalGroup *>(group);
  return g ? static_cast<void *>(g->stream) : nullptr;
}

int mpb_comm_create_local(void *group, int rank, mpb_comm **out) {
  LocalGroup *g = static_cast<LocalGroup *>(group);
  if (!g || !out || rank < 0 || rank >= g->nranks) return MPB_ERR_ARG;
  mpb_comm *c = new mpb_comm();
  c->comm = nullptr;
  c->rank = rank;
  c->nranks = g->nranks;
  c->grp = g;
  *out = c;
  return MPB_OK;
}

// The end of a solve (the state is in h->h_state, the loop's events are
// recorded): final true residual, result struct, hand-over to the caller's
// stream.
static int finish_solve(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const double *b, double *x,
                        const SolveWs &w, mpb_solve_result *res, const DistCtx *dc, cudaStream_t s,
                        int64_t launches0) {
  int rc = MPB_OK;
  const unsigned nt = static_cast<unsigned>(plan->ntiles);
  const SolverState st = *h->h_state;
  if (st.error == kOk) {  // final true residual (solver.py:179-182)
    if ((rc = halo_exchange(dc, x, 8, A->n, s))) return rc;
    k_resid<true><<<persistent_grid(k_resid<true>, 0, plan->ntiles), kCtaThreads, 0, s>>>(
                                              A->sell->d_sp, A->sell->d_col, op_vals(A), plan->d_td, static_cast<int>(nt), b, x, nullptr, w.part, w.st, 0,
                                              kStepFinal, w.csum, owners_poll(plan->ntiles) ? 1 : 0);
    MPB_LAUNCHED(h);
    if ((rc = dist_step(h, dc, w.st, kStepFinal, 0, s))) return rc;
    MPB_CUDA(cudaMemcpyAsync(h->h_state, w.st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
  }
  MPB_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  MPB_CUDA(cudaEventElapsedTime(&ms, h->ev_t0, h->ev_t1));
  const SolverState fin = *h->h_state;
  res->converged = fin.converged;
  res->error = fin.error;
  res->iterations = fin.error ? fin.err_it : fin.last_it;
  res->err_iteration = fin.error ? fin.err_it : 0;
  res->err_value = fin.err_val;
  res->final_true_relres = fin.error ? NAN : fin.final_true;
  // ovf_count is global (all-reduced on the multi-GPU path); ovf_first is
  // this rank's own first local row, INT64_MAX when the overflow happened on
  // another rank (the caller all-reduces the global first index,
  // distributed.SlabSolver).  Only a row this rank owns is dereferenced.
  const bool local_ovf = fin.ovf_count && fin.ovf_first >= 0 && fin.ovf_first < A->n;
  res->overflow_count = static_cast<int64_t>(fin.ovf_count);
  res->overflow_index = local_ovf ? fin.ovf_first : -1;
  if (fin.error == kNarrowOverflow) {  // the offending r entry
    res->err_value = NAN;
    if (local_ovf)
      MPB_CUDA(cudaMemcpy(&res->err_value, w.r + fin.ovf_first, sizeof(double), cudaMemcpyDeviceToHost));
  }
  res->device_seconds = 1e-3 * ms;
  res->kernel_launches = h->launches - launches0;
  MPB_CUDA(cudaEventRecord(h->ev_out, s));
  MPB_CUDA(cudaStreamWaitEvent(h->user, h->ev_out, 0));
  return MPB_OK;
}

// ---- small problems: the whole loop in k_solve_small ------------------------
static bool small_mode(const mpb_handle *h, const mpb_plan *p, const mpb_csr *A, const mpb_solve_options *o,
                       const DistCtx *dc) {
  static const bool off = std::getenv("MPB_SMALL") && std::atoi(std::getenv("MPB_SMALL")) == 0;
  if (off || dc != nullptr || !p->dia_ok || o->true_stride != 0 || std::getenv("MPB_TIMELINE")) return false;
  if (o->kind != MPB_UNIFORM && A->ib_val32 == nullptr) return false;
  if (o->kind != MPB_FIXED_LOW && A->ib_val64 == nullptr) return false;
  if ((A->op_sell_val64 ? A->op_ib_val64 : A->ib_val64) == nullptr) return false;
  (void)h;
  // every CTA of the grid must be resident at once (cooperative launch)
  int per_sm = 0, coop = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess || !coop)
    return false;
  const size_t dyn = sizeof(double) * kTileRows * kDiaSlots * 2 + sizeof(float) * kTileRows * kDiaSlots;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_small, kCtaThreads, dyn) != cudaSuccess)
    return false;
  return per_sm >= 1 && p->ntiles <= int64_t(per_sm) * num_sms();
}

static int launch_small(mpb_handle *h, cudaStream_t s, const mpb_plan *p, const mpb_csr *A,
                        const mpb_solve_options *o, const SolveWs &w, double *x) {
  SmallArgs a{};
  a.dval32 = o->kind != MPB_UNIFORM ? A->ib_val32 + p->dia_at : nullptr;
  a.dval64 = o->kind != MPB_FIXED_LOW ? A->ib_val64 + p->dia_at : nullptr;
  a.dvalop = (A->op_sell_val64 ? A->op_ib_val64 : A->ib_val64) + p->dia_at;
  a.dmeta = p->d_dmeta;
  a.td = p->d_td;
  for (int u = 0; u < kDiaSlots; u++) a.doff[u] = p->dia_off[u];
  a.ntiles = static_cast<int>(p->ntiles);
  a.k = o->k;
  a.t = o->t;
  a.x = x;
  a.r = w.r;
  a.z = w.z64;
  a.pA = w.p;
  a.pB = w.p2;
  a.zA32 = w.zA32;
  a.zB32 = w.zB32;
  a.zA64 = w.zA64;
  a.zB64 = w.zB64;
  a.part_rz = w.part;
  a.part_pq = w.part2;
  a.part_rr = w.part3;
  a.bar = w.gcnt;
  a.st = w.st;
  MPB_CUDA(cudaMemsetAsync(w.gcnt, 0, sizeof(unsigned int), s));
  const bool two64 = a.dval64 != nullptr && a.dval64 != a.dvalop;
  const size_t dyn = sizeof(double) * kTileRows * kDiaSlots * (two64 ? 2 : 1) + sizeof(float) * kTileRows * kDiaSlots;
  int per_sm = 0;
  MPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_small, kCtaThreads, dyn));
  if (per_sm < 1 || p->ntiles > int64_t(per_sm) * num_sms()) return static_cast<int>(cudaErrorCooperativeLaunchTooLarge);
  void *args[] = {&a};
  MPB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(k_solve_small), dim3(static_cast<unsigned>(p->ntiles)),
                                       dim3(kCtaThreads), args, dyn, s));
  MPB_LAUNCHED(h);
  return MPB_OK;
}

static int solve_impl(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                      const double *b, double *x, double *tr_relres, double *tr_true, int32_t *tr_branch,
                      double *tr_time, void *workspace, int64_t workspace_bytes, mpb_solve_result *res,
                      const DistCtx *dc) {
  if (!opt) return MPB_ERR_ARG;
  if (opt->kind < MPB_UNIFORM || opt->kind > MPB_ADAPTIVE_LH) return MPB_ERR_POLICY;
  if (!A || (opt->kind != MPB_UNIFORM && !A->sell_val32)) return MPB_ERR_POLICY;
  int rc = check_sell(A, true, opt->kind != MPB_UNIFORM);
  if (rc == MPB_OK) rc = check_bound(plan, A);
  if (rc) return rc;
  if (!h || !plan || !b || !x || !tr_relres || !tr_true || !tr_branch || !tr_time || !res || !workspace)
    return MPB_ERR_ARG;
  if (plan->n != A->n) return MPB_ERR_PARTITION;
  if (opt->k < 1 || opt->t < 1) return MPB_ERR_SWEEPS;
  if (opt->max_iter < 1) return MPB_ERR_ARG;
  const int64_t ng = dc ? dc->halo.recv_lo + dc->halo.recv_hi : 0;
  SolveWs w = carve(plan, A->n, static_cast<char *>(workspace), ng);
  if (workspace_bytes < static_cast<int64_t>(w.bytes)) return MPB_ERR_WORKSPACE;
  std::memset(res, 0, sizeof(*res));
  res->overflow_index = -1;
  const int64_t launches0 = h->launches;
  MPB_CUDA(cudaSetDevice(h->device));
  // in-process slab group: every rank enqueues on the group's one stream,
  // iteration by iteration (no graph: the ranks meet at host barriers)
  const bool local = dc != nullptr && dc->comm->grp != nullptr;
  cudaStream_t s = local ? dc->comm->grp->stream : h->solve;
  const unsigned nt = static_cast<unsigned>(plan->ntiles);
  // order after the caller's pending work
  MPB_CUDA(cudaEventRecord(h->ev_in, h->user));
  MPB_CUDA(cudaStreamWaitEvent(s, h->ev_in, 0));

  SolverState init{};
  init.res_tol = opt->res_tol;
  init.adp_tol = opt->adp_tol;
  init.cap = opt->max_iter;
  init.stride = opt->true_stride;
  init.kind = opt->kind;
  init.ovf_first = INT64_MAX;
  init.tr_relres = tr_relres;
  init.tr_true = tr_true;
  init.tr_branch = tr_branch;
  init.tr_time = tr_time;
  init.dist = dc ? 1 : 0;
  static const bool timeline = std::getenv("MPB_TIMELINE") != nullptr;
  if (timeline) {  // diagnostics: per-iteration kernel timestamps (summary on stderr)
    if (h->d_tl == nullptr) MPB_CUDA(cudaMalloc(&h->d_tl, sizeof(unsigned long long) * kTlIters * kTlStride));
    std::vector<unsigned long long> t0(kTlIters * kTlStride);
    for (int i = 0; i < kTlIters * kTlStride; i++) t0[i] = (i % 4 == 0) ? ~0ull : 0ull;
    MPB_CUDA(cudaMemcpy(h->d_tl, t0.data(), sizeof(unsigned long long) * t0.size(), cudaMemcpyHostToDevice));
    init.tl = h->d_tl;
  }
  *h->h_state = init;
  MPB_CUDA(cudaMemcpyAsync(w.st, h->h_state, sizeof(SolverState), cudaMemcpyHostToDevice, s));
  // tile-claim counters start at zero (a launch gated off after prefetching
  // claims leaves its counter dirty; only the end of a solve gates so)
  MPB_CUDA(cudaMemsetAsync(h->d_ctr, 0, 16 * sizeof(unsigned int), s));
  MPB_CUDA(cudaMemsetAsync(w.part, 0xFF, sizeof(double) * plan->ntiles, s));  // every slot kPartEmpty
  MPB_CUDA(cudaMemsetAsync(w.ppart, 0xFF, sizeof(double) * (plan->ntiles + 1), s));
  k_fill<<<elt_blocks(opt->max_iter), kEltThreads, 0, s>>>(tr_true, opt->max_iter, NAN);
  MPB_LAUNCHED(h);
  if (!opt->has_x0) MPB_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * A->n, s));
  // r0 = b - A x0 (or b) and ||r0|| (solver.py:118-130)
  if (opt->has_x0) {
    if ((rc = halo_exchange(dc, x, 8, A->n, s))) return rc;
    k_resid<true><<<persistent_grid(k_resid<true>, 0, plan->ntiles), kCtaThreads, 0, s>>>(
                                              A->sell->d_sp, A->sell->d_col, op_vals(A), plan->d_td, static_cast<int>(nt), b, x, w.r, w.part, w.st, 0,
                                              kStepR0, w.csum, owners_poll(plan->ntiles) ? 1 : 0);
  } else {
    k_resid<false><<<persistent_grid(k_resid<false>, 0, plan->ntiles), kCtaThreads, 0, s>>>(
                                               A->sell->d_sp, A->sell->d_col, op_vals(A), plan->d_td, static_cast<int>(nt), b, nullptr, w.r, w.part, w.st,
                                               0, kStepR0, w.csum, owners_poll(plan->ntiles) ? 1 : 0);
  }
  MPB_LAUNCHED(h);
  if ((rc = dist_step(h, dc, w.st, kStepR0, 0, s))) return rc;
  MPB_CUDA(cudaMemcpyAsync(h->h_state, w.st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  res->r0_norm = h->h_state->r0;
  if (h->h_state->done) {  // ||r0|| == 0 (solver.py:128-130)
    res->converged = 1;
    MPB_CUDA(cudaEventRecord(h->ev_out, s));
    MPB_CUDA(cudaStreamWaitEvent(h->user, h->ev_out, 0));
    res->kernel_launches = h->launches - launches0;
    return MPB_OK;
  }

  // Small problems (every tile's CTA co-resident, offset-slot layout, no strided
  // true residuals): the whole loop in one persistent cooperative kernel
  if (small_mode(h, plan, A, opt, dc)) {
    k_scalar_start<<<1, 32, 0, s>>>(w.st);
    MPB_LAUNCHED(h);
    MPB_CUDA(cudaEventRecord(h->ev_t0, s));
    rc = launch_small(h, s, plan, A, opt, w, x);
    if (rc == MPB_OK) {
      MPB_CUDA(cudaEventRecord(h->ev_t1, s));
      MPB_CUDA(cudaMemcpyAsync(h->h_state, w.st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
      MPB_CUDA(cudaStreamSynchronize(s));
      return finish_solve(h, plan, A, b, x, w, res, dc, s, launches0);
    }
    // the device cannot hold the whole grid right now (e.g. SMs taken by another client):
    // nothing ran, the graph iteration below takes over; any other error is the caller's
    if (rc != static_cast<int>(cudaErrorCooperativeLaunchTooLarge)) return rc;
    cudaGetLastError();
  }
  // the symmetric offset-slot SpMV layout of the operator (one GPU; built once per value array)
  if (dc == nullptr) ensure_sym(h, const_cast<mpb_plan *>(plan), A, s);
  // capture G iterations once (cached across solves with the same buffers)
  int G = opt->graph_iters > 0 ? opt->graph_iters : kDefaultGraphIters;
  if (fused_mode(plan, opt, dc) && (G & 1)) G++;  // the two p buffers alternate per iteration
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  key.plan = plan;
  key.rp = A->row_ptr;
  key.sell = A->sell;
  key.v64 = A->sell_val64;
  key.vop = A->op_sell_val64;
  key.v32 = A->sell_val32;
  key.b = b;
  key.x = x;
  key.trr = tr_relres;
  key.trt = tr_true;
  key.trb = tr_branch;
  key.trw = tr_time;
  key.ws = workspace;
  key.kind = opt->kind;
  key.k = opt->k;
  key.t = opt->t;
  key.iters = G;
  key.stride = opt->true_stride;
  key.n = A->n;
  key.comm = dc ? dc->comm : nullptr;
  // one GPU: the loop over graph bodies runs on the device (a while node
  // whose condition the x/r update's scalar step clears when the solve is
  // done); multi-GPU: host-polled replays
  const bool loop = dc == nullptr && std::getenv("MPB_NO_WHILE") == nullptr;
  key.loop = loop ? 1 : 0;
  if (!local && !(h->have_graph && h->gkey == key)) {
    if (h->have_graph) {
      cudaGraphExecDestroy(h->gexec);
      h->have_graph = false;
    }
    const int64_t l0 = h->launches;
    cudaGraph_t graph = nullptr, body = nullptr;
    if (loop) {
      MPB_CUDA(cudaGraphCreate(&graph, 0));
      cudaError_t ce = cudaGraphConditionalHandleCreate(&h->cond, graph, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams np{};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h->cond;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      if (ce == cudaSuccess) ce = cudaGraphAddNode(&node, graph, nullptr, 0, &np);
      if (ce == cudaSuccess) body = np.conditional.phGraph_out[0];
      if (ce == cudaSuccess)
        ce = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      if (ce != cudaSuccess) {
        cudaGraphDestroy(graph);
        return status_of(ce);
      }
    } else {
      MPB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    }
    int crc = MPB_OK;
    for (int i = 0; i < G && crc == MPB_OK; i++) crc = enqueue_iteration(h, s, plan, A, opt, w, b, x, dc, i);
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &captured);
    if (!loop) graph = captured;
    if (crc != MPB_OK) {
      if (graph) cudaGraphDestroy(graph);
      return crc;
    }
    if (ce != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return status_of(ce);
    }
    ce = cudaGraphInstantiate(&h->gexec, graph, 0);
    cudaGraphDestroy(graph);
    MPB_CUDA(ce);
    h->graph_kernels = h->launches - l0;
    h->launches = l0;  // captured, not launched
    h->have_graph = true;
    h->gkey = key;
  }
  k_scalar_start<<<1, 32, 0, s>>>(w.st);
  MPB_LAUNCHED(h);
  MPB_CUDA(cudaEventRecord(h->ev_t0, s));
  // fused mode: the first iteration's first pass runs ahead of the graph;
  // wave mode: both its passes (the wave kernels run the later ones)
  if (wave_mode(plan, opt, dc)) {
    MPB_CUDA(cudaMemsetAsync(w.gcnt, 0, sizeof(unsigned int) * (plan->ntiles / 32 + 8), s));
    if (opt->kind == MPB_UNIFORM) {
      ApplyBufs<double> bb{w.zA64, w.zB64, w.res64, w.dg64, w.wA64, w.wB64};
      rc = launch_apply<double>(h, s, plan, A, opt->k, opt->t, w.r, nullptr, w.z64, nullptr, w.part, nullptr,
                                nullptr, w.st, 0, bb, dc);
    } else {
      ApplyBufs<float> bb{w.zA32, w.zB32, w.res32, w.dg32, w.wA32, w.wB32};
      rc = launch_apply<float>(h, s, plan, A, opt->k, opt->t, w.r, nullptr, w.z32, nullptr, w.part,
                               &w.st->ovf_count, &w.st->ovf_first, w.st, 1, bb, dc);
    }
    if (rc) return rc;
  } else if (fused_mode(plan, opt, dc) && (rc = enqueue_first_passes(h, s, plan, A, opt, w, dc))) {
    return rc;
  }
  h->h_state->cond = loop ? static_cast<unsigned long long>(h->cond) : 0ull;
  MPB_CUDA(cudaMemcpyAsync(&w.st->cond, &h->h_state->cond, sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  for (;;) {
    if (local) {
      const int64_t l0 = h->launches;
      for (int i = 0; i < G; i++)
        if ((rc = enqueue_iteration(h, s, plan, A, opt, w, b, x, dc, i))) return rc;
      h->graph_kernels = h->launches - l0;
      h->launches = l0;
    } else {
      MPB_CUDA(cudaGraphLaunch(h->gexec, s));
    }
    MPB_CUDA(cudaMemcpyAsync(h->h_state, w.st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
    MPB_CUDA(cudaStreamSynchronize(s));
    const long long ran = h->h_state->error ? h->h_state->err_it : h->h_state->last_it;
    if (loop) {  // bodies the while node ran
      h->launches += h->graph_kernels * std::max<long long>(1, (ran + G - 1) / G);
      break;
    }
    h->launches += h->graph_kernels;
    if (h->h_state->done) break;
  }
  MPB_CUDA(cudaEventRecord(h->ev_t1, s));
  MPB_CUDA(cudaMemsetAsync(h->d_ctr, 0, 16 * sizeof(unsigned int), s));
  if (timeline) {
    MPB_CUDA(cudaStreamSynchronize(s));
    std::vector<unsigned long long> t(kTlIters * kTlStride);
    MPB_CUDA(cudaMemcpy(t.data(), h->d_tl, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost));
    const long long last = std::min<long long>(h->h_state->last_it, kTlIters - 1);
    double acc[3][4] = {};  // per kernel: gap (start - previous step), body (end - start), tail (step - end),
                            // of which the last CTA's reduction + step (step - last CTA known)
    long long cnt = 0;
    std::vector<double> gaps[3];
    double ent[3] = {};
    long long ent_n = 0;  // per kernel, for the median (graph-body boundaries skew the mean)
    for (long long it = 5; it < last; it++) {
      const unsigned long long *r = &t[it * kTlStride];
      const unsigned long long prev = (&t[(it - 1) * kTlStride])[2 * 4 + 2];
      const unsigned long long stp[3] = {prev, r[0 * 4 + 2], r[1 * 4 + 2]};
      bool ok = prev != 0;
      for (int k = 0; k < 3; k++) ok = ok && r[k * 4] != ~0ull && r[k * 4 + 1] && r[k * 4 + 2];
      if (!ok) continue;
      for (int k = 0; k < 3; k++) {
        acc[k][0] += 1e-3 * double(r[k * 4] - stp[k]);
        gaps[k].push_back(1e-3 * double(r[k * 4] - stp[k]));
        if (k == 0 && r[12] != ~0ull && r[13] && r[15]) {  // last pass CTA entries relative to the previous step
          ent[0] += 1e-3 * (double(r[12]) - double(prev));
          ent[1] += 1e-3 * (double(r[13]) - double(prev));
          ent[2] += 1e-3 * (double(r[15]) - double(prev));
          ent_n++;
        }
        acc[k][1] += 1e-3 * double(r[k * 4 + 1] - r[k * 4]);
        acc[k][2] += 1e-3 * double(r[k * 4 + 2] - r[k * 4 + 1]);
        if (r[k * 4 + 3]) acc[k][3] += 1e-3 * double(r[k * 4 + 2] - r[k * 4 + 3]);
      }
      cnt++;
    }
    const char *nm[3] = {"last pass", "spmv+p", "update+first"};
    if (ent_n)
      std::fprintf(stderr, "[mpb timeline] last pass CTA entry after the previous step: first %6.2f us, last %6.2f us;"
                           " last CTA past its grid wait %6.2f us\n", ent[0] / ent_n, ent[1] / ent_n, ent[2] / ent_n);
    for (int k = 0; k < 3 && cnt; k++) {
      std::sort(gaps[k].begin(), gaps[k].end());
      std::fprintf(stderr,
                   "[mpb timeline] %-12s gap %6.2f us (median %5.2f, max %6.2f)  body %6.2f us  tail %6.2f us "
                   "(last-CTA sum+step %5.2f)  (mean of %lld iterations)\n",
                   nm[k], acc[k][0] / cnt, gaps[k][gaps[k].size() / 2], gaps[k].back(), acc[k][1] / cnt,
                   acc[k][2] / cnt, acc[k][3] / cnt, cnt);
    }
  }
  if (wave_mode(plan, opt, dc) && std::getenv("MPB_VERBOSE")) {
    unsigned int spins = 0;
    MPB_CUDA(cudaMemcpy(&spins, w.gcnt + plan->ntiles / 32 + 4, sizeof(unsigned int), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[mpb] wave: %u dependency polls in this solve\n", spins);
  }
  return finish_solve(h, plan, A, b, x, w, res, dc, s, launches0);
}

static int profile_impl(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                        int64_t ghosts, const double *b, double *x, void *workspace, int64_t workspace_bytes,
                        int branch, int reps, double *h_ms, bool dist);

int mpb_profile_iteration(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                          const double *b, double *x, void *workspace, int64_t workspace_bytes, int branch, int reps,
                          double *h_ms) {
  return profile_impl(h, plan, A, opt, 0, b, x, workspace, workspace_bytes, branch, reps, h_ms, false);
}

// the multi-GPU solve runs the unfused iteration (first pass, last pass,
// p-update, SpMV, x/r update): those are the kernels timed here
int mpb_profile_iteration_dist(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                               int64_t ghosts, const double *b, double *x, void *workspace,
                               int64_t workspace_bytes, int branch, int reps, double *h_ms) {
  return profile_impl(h, plan, A, opt, ghosts, b, x, workspace, workspace_bytes, branch, reps, h_ms, true);
}

static int profile_impl(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const mpb_solve_options *opt,
                        int64_t ghosts, const double *b, double *x, void *workspace, int64_t workspace_bytes,
                        int branch, int reps, double *h_ms, bool dist) {
  if (!opt || ghosts < 0) return MPB_ERR_ARG;
  int rc = check_sell(A, true, branch == 1);
  if (rc == MPB_OK) rc = check_bound(plan, A);
  if (rc) return rc;
  if (!h || !plan || !b || !x || !workspace || !h_ms || reps < 1) return MPB_ERR_ARG;
  SolveWs w = carve(plan, A->n, static_cast<char *>(workspace), ghosts);
  if (workspace_bytes < static_cast<int64_t>(w.bytes)) return MPB_ERR_WORKSPACE;
  cudaStream_t s = h->solve;
  MPB_CUDA(cudaEventRecord(h->ev_in, h->user));
  MPB_CUDA(cudaStreamWaitEvent(s, h->ev_in, 0));
  // a mid-solve state; the fused scalar steps keep it finite (alpha tiny)
  SolverState mid{};
  mid.res_tol = 0.0;
  mid.adp_tol = opt->adp_tol;
  mid.cap = int64_t(1) << 40;
  mid.kind = branch == 0 ? MPB_UNIFORM : MPB_FIXED_LOW;
  mid.it = 2;
  mid.last_it = 1;
  mid.first = 0;
  mid.branch = branch;
  mid.alpha = 1e-30;
  mid.upd_branch = branch;
  mid.beta = 0.5;
  mid.rho = mid.rho_prev = 1.0;
  mid.r0 = 1.0;
  mid.ovf_first = INT64_MAX;
  // trace writes of the relres step land in the workspace's spare slots
  mid.tr_relres = mid.tr_true = reinterpret_cast<double *>(w.zA64);
  mid.tr_branch = reinterpret_cast<int *>(w.zB64);
  mid.tr_time = reinterpret_cast<double *>(w.zB64) + 8;
  *h->h_state = mid;
  MPB_CUDA(cudaMemsetAsync(w.part, 0xFF, sizeof(double) * plan->ntiles, s));  // every slot kPartEmpty
  MPB_CUDA(cudaMemsetAsync(w.ppart, 0xFF, sizeof(double) * (plan->ntiles + 1), s));
  auto reset = [&]() -> cudaError_t {
    cudaError_t e = cudaMemcpyAsync(w.st, h->h_state, sizeof(SolverState), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && plan->wave_ok)  // wave kernels: group counters match the state's epoch
      e = cudaMemsetAsync(w.gcnt, 0, sizeof(unsigned int) * (plan->ntiles / 32 + 8), s);
    return e;
  };
  for (int i = 0; i < 18; i++) h_ms[i] = 0.0;  // 7: p-update; 8..15: the same, chained; 16/17: wave
  const unsigned nt = static_cast<unsigned>(plan->ntiles);
  // h_ms[slot]: one launch between two events (cold: launch latency, ramp
  // and drain included); h_ms[8 + slot]: `reps` launches back to back with
  // programmatic dependent launch, as the solve graph chains its kernels
  // (each launch's prologue overlaps the previous one's drain), per launch.
  // Within the chain the scalar steps advance the state as in a solve (the
  // mid-solve state keeps them finite; res_tol 0 keeps the launches live).
  auto timed = [&](int slot, auto &&launch) -> int {
    float total = 0.f;
    for (int r = 0; r < reps; r++) {
      MPB_CUDA(reset());
      MPB_CUDA(cudaEventRecord(h->ev_t0, s));
      int lrc = launch();
      if (lrc) return lrc;
      MPB_CUDA(cudaEventRecord(h->ev_t1, s));
      MPB_CUDA(cudaEventSynchronize(h->ev_t1));
      float ms = 0.f;
      MPB_CUDA(cudaEventElapsedTime(&ms, h->ev_t0, h->ev_t1));
      total += ms;
    }
    h_ms[slot] += total / reps;
    const int chained = slot < 8 ? 8 + slot : slot + 1;
    MPB_CUDA(reset());
    MPB_CUDA(cudaEventRecord(h->ev_t0, s));
    for (int r = 0; r < reps; r++) {
      int lrc = launch();
      if (lrc) return lrc;
    }
    MPB_CUDA(cudaEventRecord(h->ev_t1, s));
    MPB_CUDA(cudaEventSynchronize(h->ev_t1));
    float ms = 0.f;
    MPB_CUDA(cudaEventElapsedTime(&ms, h->ev_t0, h->ev_t1));
    h_ms[chained] += ms / reps;
    return MPB_OK;
  };
  // BJAC passes of the requested instance, one pass at a time
  auto run_pass = [&](int pass) -> int {
    const int k = opt->k;
    const bool first = pass == 0, last = pass == k - 1;
    auto setup = [&](auto &a, auto zA, auto zB, auto zfinal, int want) {
      a.sp = A->sell->d_sp;
      a.scol = A->sell->d_col;
      a.td = plan->d_td;
      a.ctr = claim_ctr(h, 0);
      a.meta = plan->d_meta;
      a.pat = plan->d_pat;
      a.boff = plan->d_boff;
      a.t = opt->t;
      a.r64 = w.r;
      a.st = w.st;
      a.csum = w.csum;
      a.want_branch = want;
      a.zin = first ? nullptr : ((pass - 1) & 1 ? zB : zA);
      a.zout = last ? zfinal : (pass & 1 ? zB : zA);
      a.part = last ? w.part : nullptr;
      if (!dist) {
        a.win = plan->win;
        a.win.zlen = static_cast<int>(A->n);
      }
    };
    if (branch == 0) {
      ApplyBufs<double> bb{w.zA64, w.zB64, w.res64, w.dg64, w.wA64, w.wB64};
      PassArgs<double> a{};
      setup(a, bb.zA, bb.zB, w.z64, 0);
      a.sval = A->sell_val64;
      a.ib_val = A->ib_val64;
      a.g = geom_for<double>(plan);
      bind_dia(a, plan);
      if (first && last) return launch_pass<double, true, true>(h, s, plan, a, bb);
      if (first) return launch_pass<double, true, false>(h, s, plan, a, bb);
      if (last) return launch_pass<double, false, true>(h, s, plan, a, bb);
      return launch_pass<double, false, false>(h, s, plan, a, bb);
    }
    ApplyBufs<float> bb{w.zA32, w.zB32, w.res32, w.dg32, w.wA32, w.wB32};
    PassArgs<float> a{};
    setup(a, bb.zA, bb.zB, w.z32, 1);
    a.sval = A->sell_val32;
    a.ib_val = A->ib_val32;
    a.g = geom_for<float>(plan);
    bind_dia(a, plan);
    a.ovf_count = &w.st->ovf_count;
    a.ovf_first = &w.st->ovf_first;
    if (first && last) return launch_pass<float, true, true>(h, s, plan, a, bb);
    if (first) return launch_pass<float, true, false>(h, s, plan, a, bb);
    if (last) return launch_pass<float, false, true>(h, s, plan, a, bb);
    return launch_pass<float, false, false>(h, s, plan, a, bb);
  };
  for (int pass = 0; pass < opt->k; pass++) {
    const int slot = pass == 0 ? 0 : (pass == opt->k - 1 ? 2 : 1);
    rc = timed(slot, [&]() { return run_pass(pass); });
    if (rc) return rc;
  }
  // fused mode (what the solve runs when k >= 2 on a tile plan): the SpMV
  // rebuilds p from z (no p-update kernel), the x/r update carries the next
  // first pass
  const bool fused = !dist && opt->k >= 2 && !plan->large && std::getenv("MPB_NO_FUSE") == nullptr;
  if (!dist) ensure_sym(h, const_cast<mpb_plan *>(plan), A, s);
  SpmvArgs sa = fused ? spmv_args(h, plan, A, w, w.p, w.p2) : spmv_args(h, plan, A, w);
  if (dist) sa.U = nullptr;
  const int ugrid = persistent_grid(k_update, 0, plan->ntiles);
  const int pgrid = persistent_grid(k_pupdate, 0, plan->ntiles);
  if (!fused) {
    rc = timed(7, [&]() -> int {
      k_pupdate<<<pgrid, kCtaThreads, 0, s>>>(plan->d_td, static_cast<int>(nt), w.z32, w.z64, w.p, w.st);
      MPB_LAUNCHED(h);
      return MPB_OK;
    });
    if (rc) return rc;
  }
  rc = timed(3, [&]() -> int { return launch_spmv(h, s, plan, sa, !dist); });
  if (rc) return rc;
  rc = timed(4, [&]() -> int {
    k_update<<<ugrid, kCtaThreads, 0, s>>>(plan->d_td, static_cast<int>(nt), x, w.p, w.q, w.r, w.part,
                                         w.st, w.csum, owners_poll(plan->ntiles) ? 1 : 0);
    MPB_LAUNCHED(h);
    return MPB_OK;
  });
  if (rc) return rc;
  // the fused x/r update + next first pass, when the solve uses it
  h_ms[5] = 0.0;
  if (fused) {
    rc = timed(5, [&]() -> int {
      if (branch == 0)
        return launch_update_first<double>(h, s, plan, A, opt->t, w.zA64, x, w.p2, w.q, w.r, w.part, nullptr,
                                           nullptr, w.st, 0);
      return launch_update_first<float>(h, s, plan, A, opt->t, w.zA32, x, w.p2, w.q, w.r, w.part, &w.st->ovf_count,
                                        &w.st->ovf_first, w.st, 1);
    });
    if (rc) return rc;
  }
  // the wave kernel (x/r update + first pass + the next last pass), when the solve uses it
  mpb_solve_options fo = *opt;
  fo.kind = branch == 0 ? MPB_UNIFORM : MPB_FIXED_LOW;
  const bool wave = !dist && wave_mode(plan, &fo, nullptr);
  if (wave) {
    rc = timed(16, [&]() -> int {
      if (branch == 0)
        return launch_wave<double>(h, s, plan, A, opt->t, w.zA64, w.z64, x, w.p2, w.q, w.r, w.part, w.part2, w.gcnt,
                                   nullptr, nullptr, w.st, 0);
      return launch_wave<float>(h, s, plan, A, opt->t, w.zA32, w.z32, x, w.p2, w.q, w.r, w.part, w.part2, w.gcnt,
                                &w.st->ovf_count, &w.st->ovf_first, w.st, 1);
    });
    if (rc) return rc;
  }
  for (int c = 0; c < 16; c += 8) {
    double *m = h_ms + c;
    const double passes = m[1] * (opt->k > 2 ? opt->k - 2 : 0) + m[2];
    m[6] = wave ? m[3] + h_ms[16 + c / 8]
                : (fused ? passes + m[3] + m[5] + m[7] : m[0] + passes + m[3] + m[4] + m[7]);
  }
  MPB_CUDA(cudaEventRecord(h->ev_out, s));
  MPB_CUDA(cudaStreamWaitEvent(h->user, h->ev_out, 0));
  return MPB_OK;
}

int mpb_true_relres(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, const double *x, const double *b,
                    double r0_norm, double *h_out) {
  int rc = check_sell(A, true, false);
  if (rc) return rc;
  if (!h || !plan || !x || !b || !h_out) return MPB_ERR_ARG;
  if (plan->n != A->n) return MPB_ERR_PARTITION;
  const int64_t nt = plan->ntiles;
  rc = ensure_scratch(h, al256(sizeof(double) * (nt + 1)) + chunk_scratch(sizeof(double), nt) + 256);
  if (rc) return rc;
  double *part = static_cast<double *>(h->scratch);
  double *csum = reinterpret_cast<double *>(static_cast<char *>(h->scratch) + al256(sizeof(double) * (nt + 1)));
  double *out = reinterpret_cast<double *>(reinterpret_cast<char *>(csum) + chunk_scratch(sizeof(double), nt));
  k_resid<true><<<persistent_grid(k_resid<true>, 0, nt), kCtaThreads, 0, h->user>>>(
      A->sell->d_sp, A->sell->d_col, op_vals(A), plan->d_td, static_cast<int>(nt), b, x, nullptr,
      part, nullptr, 0, kStepFinal, nullptr, 0);
  MPB_LAUNCHED(h);
  if ((rc = launch_fin<double>(h, part, nt, csum, out))) return rc;
  double v;
  MPB_CUDA(cudaMemcpyAsync(&v, out, sizeof(double), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  *h_out = std::sqrt(v) / r0_norm;
  return MPB_OK;
}

// ---- row features (features.py restated on the device) ---------------------
int mpb_row_features(mpb_handle *h, int64_t n, const int32_t *row_ptr, const int32_t *col_idx, const double *val64,
                     const float *val32, double *tau, double *dom, double *row_sum, double *abs_sum, double *diag) {
  if (!h || n < 0 || !row_ptr || !col_idx || (val64 == nullptr) == (val32 == nullptr)) return MPB_ERR_ARG;
  if (n == 0) return MPB_OK;
  MPB_CUDA(cudaSetDevice(h->device));
  if (val64)
    k_row_features<double><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, row_ptr, col_idx, val64, tau, dom, row_sum,
                                                                       abs_sum, diag);
  else
    k_row_features<float><<<elt_blocks(n), kEltThreads, 0, h->user>>>(n, row_ptr, col_idx, val32, tau, dom, row_sum,
                                                                      abs_sum, diag);
  MPB_LAUNCHED(h);
  return MPB_OK;
}

int mpb_tau_histogram(mpb_handle *h, int64_t n, const double *tau, const double *h_edges, int nedges,
                      int64_t *h_counts, int64_t *h_undefined) {
  if (!h || n < 0 || (n > 0 && !tau) || !h_edges || nedges < 1 || nedges > kMaxEdges || !h_counts || !h_undefined)
    return MPB_ERR_ARG;
  MPB_CUDA(cudaSetDevice(h->device));
  int rc = ensure_scratch(h, 2 * al256(sizeof(double) * (kMaxEdges + 1)));
  if (rc) return rc;
  unsigned long long *cnt = static_cast<unsigned long long *>(h->scratch);
  double *edges = reinterpret_cast<double *>(static_cast<char *>(h->scratch) + al256(sizeof(double) * (kMaxEdges + 1)));
  MPB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (nedges + 1), h->user));
  MPB_CUDA(cudaMemcpyAsync(edges, h_edges, sizeof(double) * nedges, cudaMemcpyHostToDevice, h->user));
  if (n > 0) {
    k_tau_histogram<<<std::min(elt_blocks(n), 4 * num_sms()), kEltThreads, 0, h->user>>>(n, tau, edges, nedges, cnt);
    MPB_LAUNCHED(h);
  }
  std::vector<unsigned long long> hc(nedges + 1);
  MPB_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(unsigned long long) * (nedges + 1), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  for (int j = 0; j < nedges; j++) h_counts[j] = static_cast<int64_t>(hc[j]);
  *h_undefined = static_cast<int64_t>(hc[nedges]);
  return MPB_OK;
}

int mpb_vector_stats(mpb_handle *h, int64_t n, const double *x, double thresh, double *h_min, double *h_median,
                     double *h_max, int64_t *h_count_gt) {
  if (!h || n < 1 || !x || !h_min || !h_median || !h_max || !h_count_gt) return MPB_ERR_ARG;
  MPB_CUDA(cudaSetDevice(h->device));
  size_t sort_bytes = 0;
  MPB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, static_cast<const double *>(nullptr),
                                          static_cast<double *>(nullptr), static_cast<int>(n)));
  const size_t acc_b = 256, vec_b = al256(sizeof(double) * n);
  int rc = ensure_scratch(h, acc_b + vec_b + al256(sort_bytes));
  if (rc) return rc;
  char *base = static_cast<char *>(h->scratch);
  unsigned long long *acc = reinterpret_cast<unsigned long long *>(base);
  double *sorted = reinterpret_cast<double *>(base + acc_b);
  void *tmp = base + acc_b + vec_b;
  const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
  MPB_CUDA(cudaMemcpyAsync(acc, init, sizeof(init), cudaMemcpyHostToDevice, h->user));
  k_vector_stats<<<std::min(elt_blocks(n), 4 * num_sms()), kEltThreads, 0, h->user>>>(n, x, thresh, acc);
  MPB_LAUNCHED(h);
  unsigned long long ha[4];
  MPB_CUDA(cudaMemcpyAsync(ha, acc, sizeof(ha), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  *h_count_gt = static_cast<int64_t>(ha[3]);
  if (ha[2]) {  // numpy: min, max and median of an array holding NaN are NaN
    *h_min = *h_max = *h_median = NAN;
    return MPB_OK;
  }
  *h_min = dkey_inv(ha[0]);
  *h_max = dkey_inv(ha[1]);
  // median (np.median: the middle value, or the mean of the middle two)
  MPB_CUDA(cub::DeviceRadixSort::SortKeys(tmp, sort_bytes, x, sorted, static_cast<int>(n), 0, 64, h->user));
  MPB_LAUNCHED(h);
  double mid[2] = {0.0, 0.0};
  const int64_t m0 = (n - 1) / 2;
  MPB_CUDA(cudaMemcpyAsync(mid, sorted + m0, sizeof(double) * (n % 2 ? 1 : 2), cudaMemcpyDeviceToHost, h->user));
  MPB_CUDA(cudaStreamSynchronize(h->user));
  *h_median = n % 2 ? mid[0] : (mid[0] + mid[1]) / 2.0;
  return MPB_OK;
}

int mpb_first_violations(mpb_handle *h, int kind, int64_t n, const double *a, const double *b, double tol,
                         const int32_t *row_ptr, int64_t nrows, const int32_t *col_idx, const double *val64,
                         const float *val32, int k, int64_t *h_idx, int64_t *h_found) {
  if (!h || n < 0 || k < 1 || k > 1024 || !h_idx || !h_found || kind < 0 || kind > 2) return MPB_ERR_ARG;
  if ((kind == 0 && !a) || (kind == 1 && (!a || !b)) ||
      (kind == 2 && (!row_ptr || !col_idx || nrows < 1 || (val64 == nullptr) == (val32 == nullptr))))
    return MPB_ERR_ARG;
  *h_found = 0;
  if (n == 0) return MPB_OK;
  MPB_CUDA(cudaSetDevice(h->device));
  constexpr int kChunkBlocks = 4096;  // items per round: 4096 * kFlagBlock
  const size_t out_b = al256(sizeof(long long) * kChunkBlocks * k), cnt_b = al256(sizeof(int) * kChunkBlocks);
  int rc = ensure_scratch(h, out_b + cnt_b);
  if (rc) return rc;
  long long *out = static_cast<long long *>(h->scratch);
  int *cnt = reinterpret_cast<int *>(static_cast<char *>(h->scratch) + out_b);
  std::vector<long long> ho(static_cast<size_t>(kChunkBlocks) * k);
  std::vector<int> hcnt(kChunkBlocks);
  int64_t found = 0;
  for (long long base = 0; base < n && found < k; base += (long long)kChunkBlocks * kFlagBlock) {
    const long long items = std::min<long long>(n - base, (long long)kChunkBlocks * kFlagBlock);
    const int blocks = static_cast<int>((items + kFlagBlock - 1) / kFlagBlock);
    if (kind == 2 && val32)
      k_first_flags<float><<<blocks, 256, 0, h->user>>>(kind, n, base, a, b, tol, row_ptr, nrows, col_idx, val32, k,
                                                        out, cnt);
    else
      k_first_flags<double><<<blocks, 256, 0, h->user>>>(kind, n, base, a, b, tol, row_ptr, nrows, col_idx, val64, k,
                                                         out, cnt);
    MPB_LAUNCHED(h);
    MPB_CUDA(cudaMemcpyAsync(hcnt.data(), cnt, sizeof(int) * blocks, cudaMemcpyDeviceToHost, h->user));
    MPB_CUDA(cudaMemcpyAsync(ho.data(), out, sizeof(long long) * blocks * k, cudaMemcpyDeviceToHost, h->user));
    MPB_CUDA(cudaStreamSynchronize(h->user));
    for (int blk = 0; blk < blocks && found < k; blk++)
      for (int j = 0; j < std::min(hcnt[blk], k) && found < k; j++) h_idx[found++] = ho[static_cast<size_t>(blk) * k + j];
  }
  *h_found = found;
  return MPB_OK;
}

