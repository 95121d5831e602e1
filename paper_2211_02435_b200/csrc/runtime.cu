// runtime.cu — context, memory and the C ABI of include/lbm.h.
//
// Host-side runtime: validates the method (admissibility),
// lays the population grid out in HBM (kernels.cuh), dispatches to the
// instantiated kernels (ops_inst.cu) and moves host data in and out.  No
// arithmetic of the method runs on the host: every population, moment and
// macroscopic value is produced by the device kernels.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <dlfcn.h>   // libnccl.so.2 is loaded at run time (the NCCL of the process if any)
#include <nccl.h>    // types only
#include <unistd.h>  // getpid: same-process peers use plain device pointers

#include <chrono>
#include <mutex>
#include <thread>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for Nsight timelines

#include "../../include/lbm.h"
#include "ops.cuh"

namespace {
struct NvtxRange {  // scoped NVTX range around the C-ABI entry points (tracing)
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using lbm::GridParams;
using lbm::Ops;

// one exported table getter per (stencil, precision, space, regime) translation unit
#define LBM_DECL_OPS(st, pr, sp)                                                     \
  extern "C" const Ops *lbm_ops_##st##_##pr##_##sp##_r0(int rs);                      \
  extern "C" const Ops *lbm_ops_##st##_##pr##_##sp##_r1(int rs);                      \
  extern "C" const Ops *lbm_ops_##st##_##pr##_##sp##_r2(int rs);                      \
  static const Ops *lbm_ops_##st##_##pr##_##sp(int regime, int rs) {                  \
    switch (regime) {                                                                 \
      case 0: return lbm_ops_##st##_##pr##_##sp##_r0(rs);                             \
      case 1: return lbm_ops_##st##_##pr##_##sp##_r1(rs);                             \
      case 2: return lbm_ops_##st##_##pr##_##sp##_r2(rs);                             \
      default: return nullptr;                                                        \
    }                                                                                 \
  }
#define LBM_DECL_ALL(st, pr)          \
  LBM_DECL_OPS(st, pr, POPULATION)    \
  LBM_DECL_OPS(st, pr, RAW)           \
  LBM_DECL_OPS(st, pr, CENTRAL)       \
  LBM_DECL_OPS(st, pr, CUMULANT)
LBM_DECL_ALL(D2Q9, f64)
LBM_DECL_ALL(D2Q9, f32)
LBM_DECL_ALL(D3Q19, f64)
LBM_DECL_ALL(D3Q19, f32)
LBM_DECL_ALL(D3Q27, f64)
LBM_DECL_ALL(D3Q27, f32)
LBM_DECL_OPS(D2Q9, f64, SWE)
LBM_DECL_OPS(D2Q9, f32, SWE)
LBM_DECL_OPS(D2Q9, f64, SWEK)
LBM_DECL_OPS(D2Q9, f32, SWEK)

namespace {

const Ops *find_ops(int stencil, int prec, int space, int regime, int rs) {
#define LBM_CASE_SPACE(st, pr)                              \
  switch (space) {                                          \
    case LBM_SPACE_POPULATION: return lbm_ops_##st##_##pr##_POPULATION(regime, rs); \
    case LBM_SPACE_RAW: return lbm_ops_##st##_##pr##_RAW(regime, rs);               \
    case LBM_SPACE_CENTRAL: return lbm_ops_##st##_##pr##_CENTRAL(regime, rs);       \
    case LBM_SPACE_CUMULANT: return lbm_ops_##st##_##pr##_CUMULANT(regime, rs);     \
    default: return nullptr;                                \
  }
  if (space == lbm::SPACE_SWE) {
    if (stencil != LBM_D2Q9) return nullptr;
    return prec == LBM_FP64 ? lbm_ops_D2Q9_f64_SWE(regime, rs) : lbm_ops_D2Q9_f32_SWE(regime, rs);
  }
  if (space == lbm::SPACE_SWE_K) {
    if (stencil != LBM_D2Q9) return nullptr;
    return prec == LBM_FP64 ? lbm_ops_D2Q9_f64_SWEK(regime, rs) : lbm_ops_D2Q9_f32_SWEK(regime, rs);
  }
  if (stencil == LBM_D2Q9) {
    if (prec == LBM_FP64) { LBM_CASE_SPACE(D2Q9, f64) } else { LBM_CASE_SPACE(D2Q9, f32) }
  } else if (stencil == LBM_D3Q19) {
    if (prec == LBM_FP64) { LBM_CASE_SPACE(D3Q19, f64) } else { LBM_CASE_SPACE(D3Q19, f32) }
  } else if (stencil == LBM_D3Q27) {
    if (prec == LBM_FP64) { LBM_CASE_SPACE(D3Q27, f64) } else { LBM_CASE_SPACE(D3Q27, f32) }
  }
  return nullptr;
#undef LBM_CASE_SPACE
}

thread_local std::string g_create_error;

// WO-MRT basis (reading R31): classical Gram-Schmidt of the
// stencil's raw-moment monomials in graded-lexicographic order (x > y > z) under the weighted
// inner product <p, r> = sum_i w_i p(xi_i) r(xi_i), polynomials kept monic in their leading
// monomial.  L[p][e]: coefficient of monomial e (cube index a + 3 b + 9 c) in polynomial p;
// Linv = L^{-1} (unit lower-triangular in that order, forward substitution).
template <class S>
void wo_basis(double *L, double *Linv) {
  std::vector<int> mono;
  for (int deg = 0; deg <= 6; ++deg)
    for (int a = 2; a >= 0; --a)
      for (int b = 2; b >= 0; --b)
        for (int cz = 2; cz >= 0; --cz)
          if (a + b + cz == deg && (S::D == 3 || cz == 0) && lbm::mono_present<S>(a + 3 * b + 9 * cz))
            mono.push_back(a + 3 * b + 9 * cz);
  const int q = S::Q, n = (int)mono.size();  // n == q
  auto value = [&](int e, int i) {
    const int ex[3] = {lbm::ex_of(e), lbm::ey_of(e), lbm::ez_of(e)};
    const int v[3] = {S::vx(i), S::vy(i), S::vz(i)};
    double r = 1;
    for (int a = 0; a < 3; ++a)
      for (int k = 0; k < ex[a]; ++k) r *= v[a];
    return r;
  };
  std::vector<double> C((size_t)n * n, 0.0), P((size_t)n * q, 0.0);  // coefficients, values
  for (int k = 0; k < n; ++k) {
    C[(size_t)k * n + k] = 1.0;
    for (int i = 0; i < q; ++i) P[(size_t)k * q + i] = value(mono[k], i);
    for (int j = 0; j < k; ++j) {
      double num = 0, den = 0;
      for (int i = 0; i < q; ++i) {
        const double w = lbm::weight<S>(i);
        num += w * value(mono[k], i) * P[(size_t)j * q + i];
        den += w * P[(size_t)j * q + i] * P[(size_t)j * q + i];
      }
      const double cf = num / den;
      for (int m = 0; m <= j; ++m) C[(size_t)k * n + m] -= cf * C[(size_t)j * n + m];
      for (int i = 0; i < q; ++i) P[(size_t)k * q + i] -= cf * P[(size_t)j * q + i];
    }
  }
  // inverse of the unit lower-triangular C
  std::vector<double> Ci((size_t)n * n, 0.0);
  for (int col = 0; col < n; ++col)
    for (int r = col; r < n; ++r) {
      double s = (r == col) ? 1.0 : 0.0;
      for (int m = col; m < r; ++m) s -= C[(size_t)r * n + m] * Ci[(size_t)m * n + col];
      Ci[(size_t)r * n + col] = s;
    }
  for (int k = 0; k < 27 * 27; ++k) L[k] = Linv[k] = 0.0;
  for (int p = 0; p < n; ++p)
    for (int m = 0; m < n; ++m) {
      L[p * 27 + mono[m]] = C[(size_t)p * n + m];     // polynomial p over cube monomials
      Linv[mono[m] * 27 + p] = Ci[(size_t)m * n + p]; // monomial m over polynomials
    }
}

// ---- NCCL, loaded at run time: the library that is already in the process (torch's) is
// preferred, so one process never mixes two NCCL builds; LBM_NCCL_LIB overrides the path.
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = nullptr;
    if (const char *path = getenv("LBM_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char *e = dlerror();
      api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](auto &fn, const char *name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    const bool all = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
                     sym(api.CommDestroy, "ncclCommDestroy") && sym(api.GroupStart, "ncclGroupStart") &&
                     sym(api.GroupEnd, "ncclGroupEnd") && sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") &&
                     sym(api.GetErrorString, "ncclGetErrorString");
    if (!all) api.err = "libnccl.so.2 lacks a required symbol";
    api.ok = all;
  });
  return api;
}

}  // namespace

struct lbm_ctx {
  int stencil = 0, space = 0, eq = 0, zc = 0, regime = 0, prec = 0, streaming = 0, kspace = 0;
  const Ops *ops = nullptr;
  int q = 0, d = 0;
  int gnx = 0, gny = 0, gnz = 0;
  int rank = 0, nranks = 1, offset = 0, extent = 0;
  int bb = 0;
  int rs = 0;
  GridParams g{};
  size_t esize = 8, grid_elems = 0;
  void *buf[2] = {nullptr, nullptr};
  int cur = 0;       // pull: index of the current grid
  int aa_state = 0;  // AA: 0 = state A, 1 = state B
  long long steps = 0;
  alignas(16) unsigned char params[sizeof(lbm::MethodParams<double>)];  // MethodParams<real>
  double rates_d[27] = {0};
  double force[3] = {0, 0, 0};
  bool forced = false;
  int force_model = LBM_FORCE_GUO;
  bool resident_failed = false;  // the cluster-resident launch was refused once: do not retry
  // two-step sweeps across ranks (peer path): 8 scratch planes behind the planes of each grid
  // (grid 0's are used: the neighbours map grid 0 anyway), element offset scratch_off
  bool peer_tb_cap = false;
  size_t scratch_off = 0;
  void *peer_scr[2] = {};  // the lower / upper neighbour's scratch (plane 0)
  int last_cluster = 0;
  const Ops *ops_plain = nullptr;  // the unforced kernels chosen at create
  bool tb_allowed = false;         // temporal blocking (two fused steps) eligible
  cudaGraphExec_t graph[2] = {nullptr, nullptr};  // captured step loops per parity (small lattices)
  double swe_g = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void *staging = nullptr;
  size_t staging_bytes = 0;
  int *flag = nullptr;
  // fused halo push between slab contexts (lbm_peer_*)
  long long *peer_flags = nullptr;      // device [2]: phases completed by the lower / upper neighbour; [2] timeout
  void *peer_ghost[2][2] = {};          // [grid][0 lower, 1 upper]: the plane the boundary kernels
                                        // address in the neighbour (pull: its ghost plane of the
                                        // next grid; AA: its adjacent boundary plane)
  void *peer_base[2][2] = {};           // [grid][side]: the neighbours' grid bases
  long long *peer_remote[2] = {};       // lower neighbour's flags[1], upper neighbour's flags[0]
  void *peer_mapped[6] = {};            // CUDA IPC mappings to close, keyed by (pid, exported pointer)
  void *peer_raw[6] = {};
  long long peer_pid[6] = {};
  int n_mapped = 0;
  cudaGraphExec_t peer_graph[2] = {nullptr, nullptr};  // captured lbm_step_peer loops per grid parity
  int peer_graph_steps = 0;                            // steps per captured loop (32 or 36)
  bool peer_on = false;
  // host-ordered waits (a neighbour shares this GPU): no kernel spins on a flag another rank
  // writes; the host polls the flags and enqueues the dependent work only once they are set
  bool peer_host_wait = false;
  long long host_phase = 0;             // signals enqueued since connect (the device's flags[3])
  bool host_timed_out = false;
  cudaStream_t s_poll = nullptr;        // D2H reads of the flags
  long long *h_flags = nullptr;         // pinned [2]
  unsigned char uuid[16] = {};          // this context's device
  cudaStream_t s_int = nullptr;         // interior planes of lbm_step_peer
  cudaEvent_t ev_b = nullptr, ev_i = nullptr;
  // slab decomposition with ghost planes (nranks > 1, or one rank exchanging with itself
  // through NCCL): the periodic wrap along the slab axis goes through the ghost planes
  bool multi = false;
  bool needs_prime = false;  // the current halo must be exchanged before the next lbm_step
  ncclComm_t comm = nullptr; // in-library NCCL halo exchange (lbm_domain.nccl_id)
  void *(*dev_alloc)(size_t, void *) = nullptr;
  void (*dev_free)(void *, void *) = nullptr;
  void *alloc_user = nullptr;
  std::string err;
};

namespace {

lbm_status fail(lbm_ctx *c, lbm_status s, const std::string &msg) {
  if (c) c->err = msg;
  else g_create_error = msg;
  return s;
}

lbm_status cuda_fail(lbm_ctx *c, cudaError_t e, const char *what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(c, e == cudaErrorMemoryAllocation ? LBM_ENOMEM : LBM_ECUDA, m);
}

#define LBM_CUDA(c, call)                                   \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail((c), e_, #call); \
  } while (0)

lbm_status check_launch(lbm_ctx *c, const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, what);
  return LBM_OK;
}

lbm_status ensure_staging(lbm_ctx *c, size_t bytes) {
  if (c->staging_bytes >= bytes) return LBM_OK;
  if (c->staging) cudaFree(c->staging);
  c->staging = nullptr;
  c->staging_bytes = 0;
  LBM_CUDA(c, cudaMalloc(&c->staging, bytes));
  c->staging_bytes = bytes;
  return LBM_OK;
}

int q_of(int stencil) { return stencil == LBM_D2Q9 ? 9 : (stencil == LBM_D3Q19 ? 19 : 27); }

long long local_cells(const lbm_ctx *c) { return (long long)c->g.nx * c->g.ny * c->g.nzl; }

void *grid_ptr(lbm_ctx *c, int which) {
  if (c->streaming != LBM_PULL) return c->buf[0];  // in place: one grid
  return c->buf[which == 0 ? c->cur : 1 - c->cur];
}

// the kernels' method parameters in the storage precision
template <class real>
void fill_params_t(lbm_ctx *c) {
  lbm::MethodParams<real> p{};
  for (int i = 0; i < 27; ++i) {
    p.rates.w[i] = (real)c->rates_d[i];
    p.force.half.w[i] = (real)(0.5 * c->rates_d[i]);
  }
  for (int a = 0; a < 3; ++a) p.force.F[a] = (real)c->force[a];
  std::memcpy(c->params, &p, sizeof(p));
}
void fill_params(lbm_ctx *c) {
  if (c->esize == 8) fill_params_t<double>(c);
  else fill_params_t<float>(c);
}

// CUDA-graph replay of the step loop for launch-bound (small) lattices
constexpr int kGraphSteps = 32;                    // even: the storage parity is unchanged
constexpr long long kGraphMaxCells = 1LL << 20;    // ~ < 50 us per step

void drop_graphs(lbm_ctx *c) {
  for (auto &gx : c->graph)
    if (gx) {
      cudaGraphExecDestroy(gx);
      gx = nullptr;
    }
  for (auto &gx : c->peer_graph)
    if (gx) {
      cudaGraphExecDestroy(gx);
      gx = nullptr;
    }
}

bool graphs_enabled() {
  const char *env = getenv("LBM_CUDA_GRAPHS");
  return !(env && env[0] == '0');
}

// two fused pull steps available for this context and its current kernels
// Temporal blocking: CTAs (tile columns x slab chunks) for >= 4 waves (148 SMs x 2 CTAs),
// slab chunks of >= 32 planes (each chunk recomputes two step-(t+1) planes).
constexpr long long kTbMinCtas = 4 * 2 * 148;
constexpr int kTbMinChunkPlanes = 32;

long long tb_tiles(const lbm_ctx *c) {
  return (long long)(c->g.nx / c->ops->tile_x) * (c->g.ny / c->ops->tile_y);
}

int tb_zchunks(const lbm_ctx *c) {
  const int n = c->g.nzl;
  if (const char *e = getenv("LBM_TB_ZCHUNKS")) {  // test hook
    const int k = atoi(e);
    return k < 1 ? 1 : (k > n ? n : k);
  }
  // twice the chunks the 4-wave minimum needs (>= 8 waves where the slab allows chunks of >= 32
  // planes): the tail of the last wave shrinks; C2 256^3 6 vs 3 chunks: fp32 52.6k vs 51.0k,
  // fp64 30.4k vs 29.9k MLUPS (profiles/r2/tb_zchunks.txt); C5 depth 3 74 vs 37 chunks: 0.73 vs
  // 0.74-0.77 ms per step (profiles/r2/tb2d_one_barrier.txt)
  const long long tiles = tb_tiles(c);
  const long long need = 2 * ((kTbMinCtas + tiles - 1) / tiles);
  const int maxch = n / kTbMinChunkPlanes > 1 ? n / kTbMinChunkPlanes : 1;
  return (int)(need < maxch ? need : maxch);
}

// two fused steps per call pair on the peer path (multi-rank): interior planes [2, nzl - 2)
// by the two-step sweep, the two boundary regions by two single steps through the scratch
bool use_peer_tb(const lbm_ctx *c) {
  return c->peer_tb_cap && (c->peer_on || c->comm) && c->streaming == LBM_PULL;
}
// three fused steps per triple across ranks (2D; fused peer push or in-library NCCL): the
// interior rows [3, nzl - 3) by the depth-3 sweep, the boundary regions by three single steps
// through the scratch planes 8..29 (enqueue_peer_steps / enqueue_nccl_steps); >= 10 rows per
// slab; LBM_TB_DEPTH=2 keeps pairs
// the context has the three-step regions (2D slab with the pair scratch, >= 10 rows, 256-cell strips)
bool tb3_cap(const lbm_ctx *c) {
  if (!c->peer_tb_cap || c->streaming != LBM_PULL || c->d != 2 || !c->ops->pull3 || c->g.nzl < 10 ||
      c->g.nx % 256 != 0)
    return false;
  const char *env = getenv("LBM_TB_DEPTH");
  return !(env && env[0] == '2');
}

bool use_peer_tb3(const lbm_ctx *c) { return use_peer_tb(c) && tb3_cap(c); }

int peer_tb_chunks(const lbm_ctx *c) {
  const long long tiles = tb_tiles(c);
  const long long need = (kTbMinCtas + tiles - 1) / tiles;
  const int maxch = (c->g.nzl - 4) / kTbMinChunkPlanes > 1 ? (c->g.nzl - 4) / kTbMinChunkPlanes : 1;
  return (int)(need < maxch ? need : maxch);
}

bool use_temporal_blocking(const lbm_ctx *c) {
  if (!(c->tb_allowed && c->ops->pull2 && c->ops->tile_x > 0 && c->g.nx % c->ops->tile_x == 0 &&
        c->g.ny % c->ops->tile_y == 0))
    return false;
  const char *env = getenv("LBM_TEMPORAL_BLOCKING");
  if (env && env[0] == '1') return true;
  // fewer CTAs than 4 waves leave the fused sweep tail-bound
  return tb_tiles(c) * tb_zchunks(c) >= kTbMinCtas;
}

// slab chunks of the depth-3 sweep: those of the two-step sweep
int tb3_zchunks(const lbm_ctx *c) { return tb_zchunks(c); }

// three fused steps per sweep (k_pullD_2d, depth 3) for 2D lattices where the two-step sweep
// is used: C5 0.73 vs 0.82 ms per step (scripts/tb2d_depth.cu).  Environment LBM_TB_DEPTH=2
// (read per call) keeps the two-step sweep.
bool use_depth3(const lbm_ctx *c) {
  if (!c->ops->pull3 || c->d != 2 || c->g.nzl < 8 || c->g.nx % 256 != 0) return false;
  const char *env = getenv("LBM_TB_DEPTH");
  if (env && env[0] == '2') return false;
  return use_temporal_blocking(c);
}

// cluster-resident loop (k_resident2): small single-rank 2D pull lattices; returns the CTAs
// per cluster (0: not used).  The largest cluster (<= 16 CTAs, one per SM) whose CTAs hold
// their rows + 2 ghost rows of both grids in shared memory and at most kResidentMaxCellsPerCta
// cells: a step is latency-bound (collision chain + DSMEM store + cluster barrier, ~1.1 us at
// 256 cells per CTA); beyond 512 cells per CTA the CUDA-graph replay of plain launches, whose
// steps spread over all SMs, is as fast (B200: 128^2 at 16 CTAs 8.6 vs 9.1 GLUPS).
// LBM_RESIDENT=0 disables, LBM_RESIDENT_CLUSTER=k caps the cluster size (read per call).
constexpr int kResidentMaxCellsPerCta = 512;
int resident_cluster(const lbm_ctx *c) {
  if (!c->ops->resident || c->resident_failed || c->multi || c->streaming != LBM_PULL) return 0;
  const char *env = getenv("LBM_RESIDENT");
  if (env && env[0] == '0') return 0;
  int cap = 16;
  if (const char *ce = getenv("LBM_RESIDENT_CLUSTER")) cap = std::max(1, atoi(ce));
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int ny = c->g.nzl, nx = c->g.nx;
  for (int C = 16; C >= 1; C /= 2) {
    if (C > cap || ny % C != 0) continue;
    const int rows = ny / C;
    if (lbm::resident_smem(c->q, nx, rows, c->esize) <= (size_t)optin && rows * nx <= kResidentMaxCellsPerCta)
      return C;
    return 0;  // fewer CTAs only hold more rows each
  }
  return 0;
}

// graph replay: small single-rank lattice on a capturable stream; LBM_CUDA_GRAPHS=0 disables
bool use_graphs(const lbm_ctx *c) {
  if (local_cells(c) > kGraphMaxCells || c->stream == nullptr || use_temporal_blocking(c)) return false;
  return graphs_enabled();
}

// kernel of the next in-place step: AA odd/even, Esoteric Pull odd/even (state 0 -> odd)
int inplace_pattern(const lbm_ctx *c, int state) {
  if (c->streaming == LBM_AA) return state == 0 ? lbm::PAT_AA_ODD : lbm::PAT_AA_EVEN;
  if (c->streaming == LBM_ESOTERIC_TWIST) return state == 0 ? lbm::PAT_TW0 : lbm::PAT_TW1;
  if (c->streaming == LBM_ESOTERIC_PUSH) return state == 0 ? lbm::PAT_ESOP_ODD : lbm::PAT_ESOP_EVEN;
  return state == 0 ? lbm::PAT_ESO_ODD : lbm::PAT_ESO_EVEN;
}
int inplace_pattern(const lbm_ctx *c) { return inplace_pattern(c, c->aa_state); }

// Captures kGraphSteps single steps starting from each storage parity (pull: current grid
// 0/1; in-place: state 0/1) into an executable graph.  Done once, on the first lbm_step call
// (so a warm-up pays it), again after lbm_set_force; capture launches nothing.
lbm_status ensure_graphs(lbm_ctx *c) {
  const GridParams g = c->g;
  for (int par = 0; par < 2; ++par) {
    if (c->graph[par]) continue;
    cudaGraph_t gr = nullptr;
    LBM_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int cur = par, st = par;
    for (int k = 0; k < kGraphSteps; ++k) {
      if (c->streaming != LBM_PULL) {
        c->ops->aa(c->buf[0], g, c->params, c->swe_g, inplace_pattern(c, st), g.nzl, c->stream);
        st ^= 1;
      } else {
        c->ops->pull(c->buf[cur], c->buf[1 - cur], g, c->params, c->swe_g, c->bb, g.nzl, c->stream);
        cur ^= 1;
      }
    }
    cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->graph[par], gr, 0);
    if (gr) cudaGraphDestroy(gr);
    if (e != cudaSuccess) {
      c->graph[par] = nullptr;
      return cuda_fail(c, e, "CUDA-graph capture of the step loop");
    }
  }
  return LBM_OK;
}

// momentum correction of the canonical post-collision state: u = (j - F/2) / rho
double3 post_shift(const lbm_ctx *c) {
  if (!c->forced) return make_double3(0, 0, 0);
  return make_double3(-0.5 * c->force[0], -0.5 * c->force[1], -0.5 * c->force[2]);
}

// ---- fused halo push: completion flags (system scope, NVLink peer memory) ----
__device__ __forceinline__ long long ld_acquire_sys(const long long *p) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(long long *p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Completion flags of a context (device, 4 x int64): [0] phase completed by the lower
// neighbour, [1] by the upper neighbour (both written remotely), [2] timeout latch, [3] this
// context's own phase.  The phase lives on the device so that the step loop is a fixed
// launch sequence (capturable in a CUDA graph).

// one thread: wait until both neighbours completed this context's phase (flags[3])
__global__ void k_peer_wait(long long *flags, unsigned long long timeout_ns) {
  if (ld_acquire_sys(flags + 2)) return;  // an earlier wait gave up: do not stall again
  const long long target = flags[3];
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(flags) < target || ld_acquire_sys(flags + 1) < target) {
    if (globaltimer() - t0 > timeout_ns) {
      st_release_sys(flags + 2, 1);
      return;
    }
    __nanosleep(256);
  }
}

// one thread: advance this context's phase and publish it to both neighbours, once this
// stream's earlier work (the boundary planes and their halo stores) is complete
__global__ void k_peer_signal(long long *flags, long long *lower, long long *upper) {
  const long long phase = flags[3] + 1;
  flags[3] = phase;
  __threadfence_system();
  st_release_sys(lower, phase);
  st_release_sys(upper, phase);
}

unsigned long long peer_timeout_ns() {
  const char *env = getenv("LBM_PEER_TIMEOUT_S");
  const double s = env ? atof(env) : 60.0;
  return (unsigned long long)((s > 0 ? s : 60.0) * 1e9);
}

// The wait before a phase: on the device (a one-thread k_peer_wait spinning on the flags,
// the deployment case of one GPU per rank) or, when a neighbour shares this GPU, on the host:
// kernels that wait on one another must not run as separate launches on ONE GPU (nothing
// guarantees they are co-scheduled; across processes the spin blocks the context switch), so
// the host polls the flags (D2H reads on a private stream) and only then enqueues the work of
// the phase.  The target is the number of signals this context has enqueued, which equals the
// device-side phase flags[3] the spinning wait reads at the same point of the stream.
void peer_wait(lbm_ctx *c, unsigned long long timeout_ns) {
  if (!c->peer_host_wait) {
    k_peer_wait<<<1, 1, 0, c->stream>>>(c->peer_flags, timeout_ns);
    return;
  }
  if (c->host_timed_out) return;  // an earlier wait gave up: do not stall again
  const long long target = c->host_phase;
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    if (cudaMemcpyAsync(c->h_flags, c->peer_flags, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->s_poll) !=
            cudaSuccess ||
        cudaStreamSynchronize(c->s_poll) != cudaSuccess) {
      c->host_timed_out = true;  // reported by lbm_peer_status like a timeout
      return;
    }
    if (c->h_flags[0] >= target && c->h_flags[1] >= target) return;
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (dt * 1e9 > (double)timeout_ns) {
      c->host_timed_out = true;
      return;
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

void peer_signal(lbm_ctx *c) {
  k_peer_signal<<<1, 1, 0, c->stream>>>(c->peer_flags, c->peer_remote[0], c->peer_remote[1]);
  ++c->host_phase;
}

// Release of the boundary kernels' stores into peer memory before the completion flag
// (kernels.cuh peer_release_cta): 1 (default) = a CTA barrier, then one system-scope fence by
// thread 0 of every CTA, so the halo stores are visible system-wide before the kernel ends
// and k_peer_signal (stream-ordered after it, with its own system fence) publishes the phase;
// 2 = a fence per thread after its stores; 0 = none (ordering by kernel completion alone).
// Environment LBM_PEER_FENCE, read per call.
int peer_fence() {
  const char *env = getenv("LBM_PEER_FENCE");
  if (!env) return 1;
  if (env[0] == '0') return 0;
  if (env[0] == '2') return 2;
  return 1;
}

void peer_release(lbm_ctx *c) {
  for (int k = 0; k < c->n_mapped; ++k) cudaIpcCloseMemHandle(c->peer_mapped[k]);
  c->n_mapped = 0;
  c->peer_on = false;
}

// Enqueues n steps with the fused halo push starting from grid 'cur' (no context state
// changes: also the body of the captured graphs).  Per step: the interior planes on s_int
// after the previous step's boundary planes; on the context stream, after the previous
// interior planes: wait for the neighbours' previous phase, the two boundary planes
// (k_pull<PEER>: local stores + halo stores into the neighbours' next grid), signal.
int pull_parity(const lbm_ctx *c) { return c->streaming == LBM_PULL ? c->cur : c->aa_state; }

int enqueue_peer_steps(lbm_ctx *c, int n, int cur) {
  const unsigned long long tmo = peer_timeout_ns();
  const int nzl = c->g.nzl;
  const bool pull = c->streaming == LBM_PULL;
  cudaEventRecord(c->ev_b, c->stream);
  cudaEventRecord(c->ev_i, c->stream);
  int t = 0;
  if (use_peer_tb3(c)) {
    // Triples t -> t+3 (2D): on s_int the depth-3 sweep of the interior rows [3, nzl - 3) (its
    // widened levels reach rows 1 .. nzl - 2 of A, no ghost data); on the context stream three
    // phases, each wait / two boundary launches / signal: step t+1 of rows {0..4} and
    // {nzl-5..nzl-1} from A into the level-1 scratch (rows -1..4 at scratch planes 8..13,
    // nzl-5..nzl at 14..19), step t+2 of rows {0..3} and {nzl-4..nzl-1} from it into the
    // level-2 scratch (rows -1..3 at 20..24, nzl-4..nzl at 25..29), step t+3 of rows {0,1,2} and
    // {nzl-3..nzl-1} from it into B.  Rows 0 and nzl-1 push their slab-crossing populations into
    // the neighbours' ghost rows of the same level (their rows nzl and -1), level 3 into their
    // ghost planes of B.  Three flag phases per triple, as three single steps.
    const long long PB = (long long)c->g.plane * (long long)c->esize;
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * c->esize;
    char *lo = static_cast<char *>(c->peer_scr[0]), *hi = static_cast<char *>(c->peer_scr[1]);
    void *l1b = scr + 8 * PB, *l1t = scr + (18 - (long long)nzl) * PB;  // row z at base + (z + 1) P
    void *l2b = scr + 20 * PB, *l2t = scr + (28 - (long long)nzl) * PB;
    for (; t + 3 <= n && n - t != 4; t += 3) {  // a remainder of 4: two pairs, not triple + single
      void *A = c->buf[cur], *B = c->buf[1 - cur];
      cudaStreamWaitEvent(c->stream, c->ev_i, 0);
      cudaStreamWaitEvent(c->s_int, c->ev_b, 0);
      GridParams gi = c->g;
      gi.zbegin = 3;
      gi.zcount = nzl - 6;
      c->ops->pull3(A, B, gi, c->params, c->swe_g, peer_tb_chunks(c), c->s_int);
      cudaEventRecord(c->ev_i, c->s_int);
      GridParams g1 = c->g;
      g1.peer_fence = peer_fence();
      // level 1: row 0 -> the lower's level-1 row nzl (its plane 19), row nzl-1 -> the upper's row -1 (plane 8)
      g1.peer_lo = lo + 19 * PB;
      g1.peer_hi = hi + 8 * PB;
      peer_wait(c, tmo);
      g1.zbegin = 0;
      c->ops->pull(A, l1b, g1, c->params, c->swe_g, c->bb, 5, c->stream);
      g1.zbegin = nzl - 5;
      c->ops->pull(A, l1t, g1, c->params, c->swe_g, c->bb, 5, c->stream);
      peer_signal(c);
      // level 2: into the lower's level-2 row nzl (plane 29) and the upper's row -1 (plane 20)
      GridParams g2 = g1;
      g2.peer_lo = lo + 29 * PB;
      g2.peer_hi = hi + 20 * PB;
      peer_wait(c, tmo);
      g2.zbegin = 0;
      c->ops->pull(l1b, l2b, g2, c->params, c->swe_g, c->bb, 4, c->stream);
      g2.zbegin = nzl - 4;
      c->ops->pull(l1t, l2t, g2, c->params, c->swe_g, c->bb, 4, c->stream);
      peer_signal(c);
      // level 3: into the neighbours' ghost planes of B
      GridParams g3 = g1;
      g3.peer_lo = c->peer_ghost[1 - cur][0];
      g3.peer_hi = c->peer_ghost[1 - cur][1];
      peer_wait(c, tmo);
      g3.zbegin = 0;
      c->ops->pull(l2b, B, g3, c->params, c->swe_g, c->bb, 3, c->stream);
      g3.zbegin = nzl - 3;
      c->ops->pull(l2t, B, g3, c->params, c->swe_g, c->bb, 3, c->stream);
      peer_signal(c);
      cudaEventRecord(c->ev_b, c->stream);
      cur ^= 1;
    }
  }
  if (use_peer_tb(c)) {
    // Pairs of steps t -> t+2 (A = current grid, B = next): on s_int the two-step sweep of
    // the interior planes [2, nzl - 2) (its step-(t+1) halo planes 1 and nzl - 2 are recomputed
    // from A's own planes: no ghost data, no neighbour dependence); on the context stream:
    // wait, step t+1 of the boundary regions {0,1,2} and {nzl-3,..,nzl-1} from A into the
    // scratch (planes -1..2 and nzl-3..nzl of scratch planes 0..3 / 4..7; planes 0 and nzl-1
    // push their slab-crossing populations into the neighbours' scratch ghost planes), signal,
    // wait, step t+2 of planes {0,1} and {nzl-2,nzl-1} from the scratch into B (pushing into
    // the neighbours' ghost planes of B), signal.  Two phases per pair, as two single steps.
    const size_t PB = (size_t)c->g.plane * c->esize;
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * c->esize;
    void *s_lo = scr;                                          // plane z at scr + (z + 1) P
    void *s_hi = scr - (long long)(nzl - 6) * (long long)PB;   // plane nzl-3 at scratch plane 4
    void *nb_lo7 = static_cast<char *>(c->peer_scr[0]) + 7 * PB;  // lower's scratch plane 7
    void *nb_hi0 = c->peer_scr[1];                                // upper's scratch plane 0
    for (; t + 2 <= n; t += 2) {
      void *A = c->buf[cur], *B = c->buf[1 - cur];
      cudaStreamWaitEvent(c->stream, c->ev_i, 0);
      cudaStreamWaitEvent(c->s_int, c->ev_b, 0);
      GridParams gi = c->g;
      gi.zbegin = 2;
      gi.zcount = nzl - 4;
      c->ops->pull2(A, B, gi, c->params, c->swe_g, peer_tb_chunks(c), c->s_int);
      cudaEventRecord(c->ev_i, c->s_int);
      peer_wait(c, tmo);
      GridParams g1 = c->g;
      g1.peer_lo = nb_lo7;
      g1.peer_hi = nb_hi0;
      g1.peer_fence = peer_fence();
      g1.zbegin = 0;
      c->ops->pull(A, s_lo, g1, c->params, c->swe_g, c->bb, 3, c->stream);
      g1.zbegin = nzl - 3;
      c->ops->pull(A, s_hi, g1, c->params, c->swe_g, c->bb, 3, c->stream);
      peer_signal(c);
      peer_wait(c, tmo);
      GridParams g2 = c->g;
      g2.peer_lo = c->peer_ghost[1 - cur][0];
      g2.peer_hi = c->peer_ghost[1 - cur][1];
      g2.peer_fence = peer_fence();
      g2.zbegin = 0;
      c->ops->pull(s_lo, B, g2, c->params, c->swe_g, c->bb, 2, c->stream);
      g2.zbegin = nzl - 2;
      c->ops->pull(s_hi, B, g2, c->params, c->swe_g, c->bb, 2, c->stream);
      peer_signal(c);
      cudaEventRecord(c->ev_b, c->stream);
      cur ^= 1;
    }
  }
  for (; t < n; ++t) {
    // pull: cur = current grid; in place (AA): cur = state (0: the odd kernel runs)
    const int pat = pull ? 0 : inplace_pattern(c, cur);
    auto launch = [&](GridParams g, int z0, int np, cudaStream_t s) {
      g.zbegin = z0;
      if (pull)
        c->ops->pull(c->buf[cur], c->buf[1 - cur], g, c->params, c->swe_g, c->bb, np, s);
      else
        c->ops->aa(c->buf[0], g, c->params, c->swe_g, pat, np, s);
    };
    cudaStreamWaitEvent(c->stream, c->ev_i, 0);  // interior of the previous step
    cudaStreamWaitEvent(c->s_int, c->ev_b, 0);   // boundary of the previous step
    launch(c->g, 1, nzl - 2, c->s_int);
    cudaEventRecord(c->ev_i, c->s_int);
    peer_wait(c, tmo);
    GridParams gb = c->g;
    if (pull || pat == lbm::PAT_AA_ODD) {  // the even AA step touches only its own cells
      const int b = pull ? 1 - cur : 0;
      gb.peer_lo = c->peer_ghost[b][0];
      gb.peer_hi = c->peer_ghost[b][1];
      gb.peer_fence = peer_fence();
    }
    launch(gb, 0, 1, c->stream);
    if (nzl > 1) launch(gb, nzl - 1, 1, c->stream);
    peer_signal(c);
    cudaEventRecord(c->ev_b, c->stream);
    cur ^= 1;
  }
  cudaStreamWaitEvent(c->stream, c->ev_i, 0);
  return cur;  // the grid (pull) / state (in place) the steps end on
}

// In-place (AA) peer mode after an odd step (state B): the canonical post-collision values of
// this slab's boundary cells that cross the cut were written straight into the neighbours'
// boundary planes; copy them back into the ghost planes, where the canonical readers
// (kernels.cuh Canon) look for them.  Stream-ordered after this rank's last step; the
// neighbours must not have started their next step (ranks read in lock-step).
lbm_status peer_refresh(lbm_ctx *c) {
  if (!c->peer_on || c->streaming == LBM_PULL || c->aa_state != 1) return LBM_OK;
  lbm_layout lay;
  lbm_status s = lbm_grid_layout((lbm_stencil)c->stencil, (lbm_precision)c->prec, c->gnx, c->gny, c->gnz,
                                 c->nranks, &lay);
  if (s != LBM_OK) return fail(c, s, "layout");
  const size_t E = c->esize, bytes = lay.halo_elems * E;
  char *mine = static_cast<char *>(c->buf[0]);
  const char *lo = static_cast<const char *>(c->peer_base[0][0]);
  const char *hi = static_cast<const char *>(c->peer_base[0][1]);
  // ghost plane 0 <- the lower neighbour's last plane (slab component -1 block); ghost plane
  // nzl + 1 <- the upper neighbour's first plane (+1 block): the "post" blocks of lbm_get_halo
  LBM_CUDA(c, cudaMemcpyAsync(mine + lay.aa_post_send_lo * E, lo + lay.aa_post_recv_hi * E, bytes,
                              cudaMemcpyDefault, c->stream));
  LBM_CUDA(c, cudaMemcpyAsync(mine + lay.aa_post_send_hi * E, hi + lay.aa_post_recv_lo * E, bytes,
                              cudaMemcpyDefault, c->stream));
  return LBM_OK;
}

// ---- in-library NCCL halo exchange (lbm_domain.nccl_id) ----
// The four halo blocks of lbm_get_halo(which) with the pull grid 'grid' as the current one
// (pull: which 0 = grid 'grid', 1 = the other grid, 2 = the scratch of the two-step regions;
// in place: the single grid, which 0 = pre-odd, 1 = post-odd): send_lo, send_hi, recv_lo, recv_hi.
void halo_blocks(lbm_ctx *c, const lbm_layout &lay, int which, int grid, char *p[4]) {
  const size_t E = c->esize;
  size_t o[4] = {lay.send_lo, lay.send_hi, lay.recv_lo, lay.recv_hi};
  if (which == 3 || which == 4) {  // level-1 / level-2 scratch rows of the triples (2D)
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * E;
    const long long P = c->g.plane, nzl = c->g.nzl;
    const long long bot = which == 3 ? 8 * P : 20 * P;                      // row z at + (z + 1) P
    const long long top = which == 3 ? (18 - nzl) * P : (28 - nzl) * P;
    p[0] = scr + (bot + (long long)o[0]) * (long long)E;
    p[1] = scr + (top + (long long)o[1]) * (long long)E;
    p[2] = scr + (bot + (long long)o[2]) * (long long)E;
    p[3] = scr + (top + (long long)o[3]) * (long long)E;
    return;
  }
  if (which == 2) {
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * E;
    const size_t shift = (size_t)(c->g.nzl - 6) * (size_t)c->g.plane;
    p[0] = scr + o[0] * E;
    p[1] = scr + (o[1] - shift) * E;
    p[2] = scr + o[2] * E;
    p[3] = scr + (o[3] - shift) * E;
    return;
  }
  char *base;
  if (c->streaming == LBM_PULL) {
    base = static_cast<char *>(c->buf[which == 0 ? grid : 1 - grid]);
  } else {
    base = static_cast<char *>(c->buf[0]);
    const size_t pre[4] = {lay.aa_pre_send_lo, lay.aa_pre_send_hi, lay.aa_pre_recv_lo, lay.aa_pre_recv_hi};
    const size_t post[4] = {lay.aa_post_send_lo, lay.aa_post_send_hi, lay.aa_post_recv_lo, lay.aa_post_recv_hi};
    for (int k = 0; k < 4; ++k) o[k] = (which == 0) ? pre[k] : post[k];
  }
  for (int k = 0; k < 4; ++k) p[k] = base + o[k] * E;
}

// One halo exchange: send_hi -> upper neighbour's recv_lo, send_lo -> lower's recv_hi, in one
// NCCL group on stream s (zero-copy: the blocks are contiguous in the grid).  Per pair of
// ranks the k-th send matches the k-th receive, which also covers 2 ranks (lower = upper)
// and one rank (itself: the periodic wrap).
lbm_status nccl_exchange(lbm_ctx *c, const lbm_layout &lay, int which, int grid, cudaStream_t s) {
  const NcclApi &nc = nccl_api();
  char *p[4];
  halo_blocks(c, lay, which, grid, p);
  const ncclDataType_t t = c->esize == 8 ? ncclFloat64 : ncclFloat32;
  const size_t n = lay.halo_elems;
  const int lo = (c->rank + c->nranks - 1) % c->nranks, hi = (c->rank + 1) % c->nranks;
  ncclResult_t r = nc.GroupStart();
  if (r != ncclSuccess) return fail(c, LBM_ENCCL, std::string("ncclGroupStart: ") + nc.GetErrorString(r));
  r = nc.Send(p[1], n, t, hi, c->comm, s);
  if (r == ncclSuccess) r = nc.Recv(p[2], n, t, lo, c->comm, s);
  if (r == ncclSuccess) r = nc.Send(p[0], n, t, lo, c->comm, s);
  if (r == ncclSuccess) r = nc.Recv(p[3], n, t, hi, c->comm, s);
  const ncclResult_t r2 = nc.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return fail(c, LBM_ENCCL, std::string("NCCL halo exchange: ") + nc.GetErrorString(r));
  return LBM_OK;
}

// n steps with the NCCL exchange from grid / state 'cur' (the lbm_step_peer sequence with an
// NCCL group in place of the pushes and flags): per step the interior planes on s_int, the two
// boundary planes and the exchange on the context stream; pairs of steps for pull contexts
// with two-step sweeps (two exchanges per pair: the scratch halo, then the next grid's).
lbm_status enqueue_nccl_steps(lbm_ctx *c, int n, int &cur) {
  lbm_layout lay;
  lbm_status s = lbm_grid_layout((lbm_stencil)c->stencil, (lbm_precision)c->prec, c->gnx, c->gny, c->gnz,
                                 c->nranks, &lay);
  if (s != LBM_OK) return fail(c, s, "layout");
  const int nzl = c->g.nzl;
  const bool pull = c->streaming == LBM_PULL;
  if (c->needs_prime) {  // the current halo (pull: grid cur; in place: the pre-odd blocks)
    if ((s = nccl_exchange(c, lay, 0, cur, c->stream)) != LBM_OK) return s;
    c->needs_prime = false;
  }
  LBM_CUDA(c, cudaEventRecord(c->ev_b, c->stream));
  LBM_CUDA(c, cudaEventRecord(c->ev_i, c->stream));
  int t = 0;
  if (use_peer_tb3(c)) {  // triples (2D): as enqueue_peer_steps, an exchange after each level
    const long long PB = (long long)c->g.plane * (long long)c->esize;
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * c->esize;
    void *l1b = scr + 8 * PB, *l1t = scr + (18 - (long long)nzl) * PB;
    void *l2b = scr + 20 * PB, *l2t = scr + (28 - (long long)nzl) * PB;
    for (; t + 3 <= n && n - t != 4; t += 3) {  // a remainder of 4: two pairs, not triple + single
      void *A = c->buf[cur], *B = c->buf[1 - cur];
      cudaStreamWaitEvent(c->stream, c->ev_i, 0);
      cudaStreamWaitEvent(c->s_int, c->ev_b, 0);
      GridParams gi = c->g;
      gi.zbegin = 3;
      gi.zcount = nzl - 6;
      c->ops->pull3(A, B, gi, c->params, c->swe_g, peer_tb_chunks(c), c->s_int);
      cudaEventRecord(c->ev_i, c->s_int);
      GridParams gb = c->g;
      gb.zbegin = 0;
      c->ops->pull(A, l1b, gb, c->params, c->swe_g, c->bb, 5, c->stream);
      gb.zbegin = nzl - 5;
      c->ops->pull(A, l1t, gb, c->params, c->swe_g, c->bb, 5, c->stream);
      if ((s = nccl_exchange(c, lay, 3, cur, c->stream)) != LBM_OK) return s;
      gb.zbegin = 0;
      c->ops->pull(l1b, l2b, gb, c->params, c->swe_g, c->bb, 4, c->stream);
      gb.zbegin = nzl - 4;
      c->ops->pull(l1t, l2t, gb, c->params, c->swe_g, c->bb, 4, c->stream);
      if ((s = nccl_exchange(c, lay, 4, cur, c->stream)) != LBM_OK) return s;
      gb.zbegin = 0;
      c->ops->pull(l2b, B, gb, c->params, c->swe_g, c->bb, 3, c->stream);
      gb.zbegin = nzl - 3;
      c->ops->pull(l2t, B, gb, c->params, c->swe_g, c->bb, 3, c->stream);
      if ((s = nccl_exchange(c, lay, 1, cur, c->stream)) != LBM_OK) return s;
      cudaEventRecord(c->ev_b, c->stream);
      cur ^= 1;
      c->steps += 3;
    }
  }
  if (use_peer_tb(c)) {
    const size_t PB = (size_t)c->g.plane * c->esize;
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * c->esize;
    void *s_lo = scr, *s_hi = scr - (long long)(nzl - 6) * (long long)PB;
    for (; t + 2 <= n; t += 2) {
      void *A = c->buf[cur], *B = c->buf[1 - cur];
      cudaStreamWaitEvent(c->stream, c->ev_i, 0);
      cudaStreamWaitEvent(c->s_int, c->ev_b, 0);
      GridParams gi = c->g;
      gi.zbegin = 2;
      gi.zcount = nzl - 4;
      c->ops->pull2(A, B, gi, c->params, c->swe_g, peer_tb_chunks(c), c->s_int);
      cudaEventRecord(c->ev_i, c->s_int);
      GridParams gb = c->g;
      gb.zbegin = 0;
      c->ops->pull(A, s_lo, gb, c->params, c->swe_g, c->bb, 3, c->stream);
      gb.zbegin = nzl - 3;
      c->ops->pull(A, s_hi, gb, c->params, c->swe_g, c->bb, 3, c->stream);
      if ((s = nccl_exchange(c, lay, 2, cur, c->stream)) != LBM_OK) return s;
      gb.zbegin = 0;
      c->ops->pull(s_lo, B, gb, c->params, c->swe_g, c->bb, 2, c->stream);
      gb.zbegin = nzl - 2;
      c->ops->pull(s_hi, B, gb, c->params, c->swe_g, c->bb, 2, c->stream);
      if ((s = nccl_exchange(c, lay, 1, cur, c->stream)) != LBM_OK) return s;
      cudaEventRecord(c->ev_b, c->stream);
      cur ^= 1;
      c->steps += 2;
    }
  }
  for (; t < n; ++t) {
    const int pat = pull ? 0 : inplace_pattern(c, cur);
    auto launch = [&](int z0, int np, cudaStream_t st) {
      GridParams g = c->g;
      g.zbegin = z0;
      if (pull) c->ops->pull(c->buf[cur], c->buf[1 - cur], g, c->params, c->swe_g, c->bb, np, st);
      else c->ops->aa(c->buf[0], g, c->params, c->swe_g, pat, np, st);
    };
    cudaStreamWaitEvent(c->stream, c->ev_i, 0);  // interior of the previous step
    cudaStreamWaitEvent(c->s_int, c->ev_b, 0);   // boundary + exchange of the previous step
    launch(1, nzl - 2, c->s_int);
    cudaEventRecord(c->ev_i, c->s_int);
    launch(0, 1, c->stream);
    if (nzl > 1) launch(nzl - 1, 1, c->stream);
    // pull: the next grid's halo; in place: after the odd step the post-odd blocks return,
    // after the even step the pre-odd blocks of the next (odd) step go out
    const int which = pull ? 1 : (cur == 0 ? 1 : 0);
    if ((s = nccl_exchange(c, lay, which, cur, c->stream)) != LBM_OK) return s;
    cudaEventRecord(c->ev_b, c->stream);
    cur ^= 1;
    c->steps += 1;
  }
  LBM_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_i, 0));
  return check_launch(c, "lbm_step (NCCL exchange)");
}

}  // namespace

extern "C" {

lbm_status lbm_nccl_get_unique_id(void *out128) {
  if (!out128) return fail(nullptr, LBM_EINVAL, "out128 is NULL");
  const NcclApi &nc = nccl_api();
  if (!nc.ok) return fail(nullptr, LBM_ENCCL, nc.err);
  ncclUniqueId id;
  const ncclResult_t r = nc.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, LBM_ENCCL, std::string("ncclGetUniqueId: ") + nc.GetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return LBM_OK;
}

const char *lbm_version(void) { return "lbm-b200 0.1 (sm_100a; arXiv 2211.02435 hot path)"; }

const char *lbm_last_error(const lbm_ctx *ctx) {
  if (!ctx) return g_create_error.c_str();
  return ctx->err.c_str();
}

lbm_status lbm_slab_extent(int extent, int rank, int nranks, int *offset, int *local_extent) {
  if (!offset || !local_extent) return LBM_EINVAL;
  if (nranks < 1 || rank < 0 || rank >= nranks || extent < 1) return LBM_EINVAL;
  if (extent % nranks != 0) return LBM_EINVAL;
  const int n = extent / nranks;
  *offset = rank * n;
  *local_extent = n;
  return LBM_OK;
}

lbm_status lbm_grid_layout(lbm_stencil stencil, lbm_precision precision, int nx, int ny, int nz, int nranks,
                           lbm_layout *out) {
  if (!out) return LBM_EINVAL;
  if (stencil < LBM_D2Q9 || stencil > LBM_D3Q27) return LBM_EINVAL;
  if (precision != LBM_FP64 && precision != LBM_FP32) return LBM_EINVAL;
  if (nx < 1 || ny < 1 || nz < 1 || nranks < 1) return LBM_EINVAL;
  const bool two_d = (stencil == LBM_D2Q9);
  const int slab = two_d ? ny : nz;
  if (slab % nranks != 0) return LBM_EINVAL;
  const int nzl = slab / nranks;
  const size_t esize = (precision == LBM_FP64) ? 8 : 4;
  const size_t align = 128 / esize;
  const int q = q_of(stencil);
  out->pitch = ((size_t)nx + align - 1) / align * align;
  out->pop = (size_t)(two_d ? 1 : ny) * out->pitch;
  out->plane = (size_t)q * out->pop;
  out->planes = (size_t)nzl + 2;
  out->elements = out->planes * out->plane;
  int up0, nup;
  if (stencil == LBM_D2Q9) { up0 = lbm::D2Q9::UP0; nup = lbm::D2Q9::NUP; }
  else if (stencil == LBM_D3Q19) { up0 = lbm::D3Q19::UP0; nup = lbm::D3Q19::NUP; }
  else { up0 = lbm::D3Q27::UP0; nup = lbm::D3Q27::NUP; }
  const size_t UP = (size_t)up0 * out->pop, DN = (size_t)(up0 + nup) * out->pop;
  const size_t z0 = 0, z1 = out->plane, zn = (size_t)nzl * out->plane, zt = (size_t)(nzl + 1) * out->plane;
  // pull: the next grid's boundary planes feed the neighbours' ghost planes
  out->send_lo = z1 + DN;
  out->send_hi = zn + UP;
  out->recv_lo = z0 + UP;
  out->recv_hi = zt + DN;
  // AA, before the odd step: the boundary planes' slots the neighbours' odd step reads
  out->aa_pre_send_lo = z1 + UP;
  out->aa_pre_send_hi = zn + DN;
  out->aa_pre_recv_lo = z0 + DN;
  out->aa_pre_recv_hi = zt + UP;
  // AA, after the odd step: what this slab's boundary cells wrote into the ghost planes
  // goes back to the neighbours' boundary planes
  out->aa_post_send_lo = z0 + DN;
  out->aa_post_send_hi = zt + UP;
  out->aa_post_recv_lo = z1 + UP;
  out->aa_post_recv_hi = zn + DN;
  out->halo_elems = (size_t)nup * out->pop;
  return LBM_OK;
}

lbm_status lbm_stencil_info(lbm_stencil stencil, int *q, int *xi, int *opposite) {
  if (!q) return LBM_EINVAL;
  auto fill = [&](auto S) {
    using St = decltype(S);
    *q = St::Q;
    for (int i = 0; i < St::Q; ++i) {
      if (xi) {
        xi[3 * i + 0] = St::vx(i);
        xi[3 * i + 1] = St::vy(i);
        xi[3 * i + 2] = St::vz(i);
      }
      if (opposite) opposite[i] = St::opp(i);
    }
  };
  switch (stencil) {
    case LBM_D2Q9: fill(lbm::D2Q9{}); return LBM_OK;
    case LBM_D3Q19: fill(lbm::D3Q19{}); return LBM_OK;
    case LBM_D3Q27: fill(lbm::D3Q27{}); return LBM_OK;
    default: return LBM_EINVAL;
  }
}

lbm_status lbm_create(lbm_stencil stencil, lbm_space collision_space, lbm_equilibrium equilibrium,
                      const double *relaxation_rates, int n_rates, const lbm_domain *domain, int zero_centered,
                      lbm_ctx **out) {
  if (!out) return fail(nullptr, LBM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!domain) return fail(nullptr, LBM_EINVAL, "domain is NULL");
  if (!relaxation_rates) return fail(nullptr, LBM_EINVAL, "relaxation_rates is NULL");
  if (stencil < LBM_D2Q9 || stencil > LBM_D3Q27) return fail(nullptr, LBM_EINVAL, "unknown stencil");
  if (collision_space < LBM_SPACE_POPULATION || collision_space > LBM_SPACE_RAW_WO)
    return fail(nullptr, LBM_EINVAL, "unknown collision space");
  if (equilibrium < LBM_EQ_ABSOLUTE || equilibrium > LBM_EQ_ABSOLUTE_F0)
    return fail(nullptr, LBM_EINVAL, "unknown equilibrium");
  const int zc = zero_centered ? 1 : 0;
  const bool delta_eq = equilibrium == LBM_EQ_DELTA || equilibrium == LBM_EQ_DISCRETE_DELTA;
  const bool discrete_eq = equilibrium == LBM_EQ_DISCRETE || equilibrium == LBM_EQ_DISCRETE_DELTA;
  const bool popbg = equilibrium == LBM_EQ_ABSOLUTE_F0;        // reading R30
  const bool wo = collision_space == LBM_SPACE_RAW_WO;          // reading R31
  if (popbg && !zc)
    return fail(nullptr, LBM_EUNSUPPORTED,
                "LBM_EQ_ABSOLUTE_F0 adds the background f0 to zero-centered populations: zero_centered = 1");
  if (wo && (discrete_eq || equilibrium == LBM_EQ_SWE))
    return fail(nullptr, LBM_EUNSUPPORTED, "the WO-MRT basis is provided with the continuous equilibrium");
  // admissibility
  if (delta_eq && !zc)
    return fail(nullptr, LBM_EUNSUPPORTED, "delta equilibrium requires zero-centered storage (PAPER.md:546)");
  if (delta_eq && collision_space == LBM_SPACE_CUMULANT)
    return fail(nullptr, LBM_EUNSUPPORTED,
                "cumulant space is incompatible with the delta equilibrium (PAPER.md:430-431, 547)");
  if (equilibrium == LBM_EQ_SWE &&
      !(stencil == LBM_D2Q9 && (collision_space == LBM_SPACE_CENTRAL || collision_space == LBM_SPACE_CUMULANT)))
    return fail(nullptr, LBM_EUNSUPPORTED,
                "the shallow-water methods are provided for D2Q9, central moments (Zhou equilibrium) or "
                "cumulants (Maxwellian with cs2 = g h / 2)");
  const int q = q_of(stencil);
  const int need = (collision_space == LBM_SPACE_POPULATION) ? 1 : q;
  if (n_rates != need)
    return fail(nullptr, LBM_EINVAL, "n_rates must be " + std::to_string(need) + " for this method");
  for (int i = 0; i < n_rates; ++i)
    if (!std::isfinite(relaxation_rates[i]) || relaxation_rates[i] < 0.0 || relaxation_rates[i] > 2.0)
      return fail(nullptr, LBM_EINVAL, "relaxation rate " + std::to_string(i) + " outside [0, 2]");
  const lbm_domain &D = *domain;
  const bool two_d = (stencil == LBM_D2Q9);
  if (D.nx < 4 || D.ny < 4 || (two_d ? D.nz != 1 : D.nz < 4))
    return fail(nullptr, LBM_EINVAL, two_d ? "D2Q9 needs nx, ny >= 4 and nz == 1" : "extents must be >= 4");
  for (int a = 0; a < 3; ++a) {
    for (int s = 0; s < 2; ++s)
      if (D.bc[a][s] != LBM_BC_PERIODIC && D.bc[a][s] != LBM_BC_NOSLIP)
        return fail(nullptr, LBM_EINVAL, "unknown boundary condition");
    if ((D.bc[a][0] == LBM_BC_PERIODIC) != (D.bc[a][1] == LBM_BC_PERIODIC))
      return fail(nullptr, LBM_EINVAL, "periodic must be set on both faces of an axis");
  }
  if (D.precision != LBM_FP64 && D.precision != LBM_FP32) return fail(nullptr, LBM_EINVAL, "unknown precision");
  if (D.streaming != LBM_PULL && D.streaming != LBM_AA && D.streaming != LBM_ESOTERIC_PULL &&
      D.streaming != LBM_ESOTERIC_TWIST && D.streaming != LBM_ESOTERIC_PUSH)
    return fail(nullptr, LBM_EINVAL, "unknown streaming");
  if (D.nranks < 1 || D.rank < 0 || D.rank >= D.nranks) return fail(nullptr, LBM_EINVAL, "bad rank/nranks");
  const int slab_extent = two_d ? D.ny : D.nz;
  if (slab_extent % D.nranks != 0)
    return fail(nullptr, LBM_EINVAL, "nranks must divide the slab-axis extent");
  if (slab_extent / D.nranks < 2) return fail(nullptr, LBM_EINVAL, "slabs need at least 2 planes");
  bool any_wall = false;
  for (int a = 0; a < 3; ++a) any_wall |= (D.bc[a][0] == LBM_BC_NOSLIP);
  // ghost planes along the slab axis: several ranks, or one rank exchanging with itself
  const bool multi = D.nranks > 1 || D.nccl_id != nullptr;
  if (D.streaming == LBM_AA && any_wall && multi)
    return fail(nullptr, LBM_EUNSUPPORTED, "AA streaming with no-slip faces is provided for a single rank");
  if ((D.streaming == LBM_ESOTERIC_PULL || D.streaming == LBM_ESOTERIC_TWIST || D.streaming == LBM_ESOTERIC_PUSH) &&
      (any_wall || multi))
    return fail(nullptr, LBM_EUNSUPPORTED,
                "Esoteric Pull / Push / Twist are provided for a single rank with periodic faces");
  if ((D.dev_alloc == nullptr) != (D.dev_free == nullptr))
    return fail(nullptr, LBM_EINVAL, "dev_alloc and dev_free must be given together");

  int regime = lbm::REG_ABS;
  if (zc) regime = delta_eq ? lbm::REG_DELTA : lbm::REG_ZC_ABS;  // ABSOLUTE_F0: REG_ZC_ABS + RS_POPBG
  int kspace = wo ? (int)LBM_SPACE_RAW : (int)collision_space;
  if (equilibrium == LBM_EQ_SWE)
    kspace = (collision_space == LBM_SPACE_CUMULANT) ? (int)lbm::SPACE_SWE_K : (int)lbm::SPACE_SWE;
  // rate specialisation: rates equal to one become compile-time constants
  int rs = lbm::RS_GENERAL;
  if (collision_space != LBM_SPACE_POPULATION) {
    const char *env = getenv("LBM_RATE_SPECIALIZATION");
    const bool allow = !(env && env[0] == '0');
    const int first_nonshear = (stencil == LBM_D2Q9) ? 5 : 9;
    bool reg = true, high = (stencil == LBM_D3Q27);
    for (int i = first_nonshear; i < q; ++i) reg &= (relaxation_rates[i] == 1.0);
    if (high)
      for (int i = 23; i < 27; ++i) high &= (relaxation_rates[i] == 1.0);
    if (allow) rs = reg ? lbm::RS_REG : (high ? lbm::RS_HIGH : lbm::RS_GENERAL);
  }
  if (discrete_eq) rs = lbm::RS_GENERAL | lbm::RS_DISCRETE;  // q_eq = T(f_eq), general rates
  if (wo || popbg)  // general rates (no rate specialisation) with the basis / background flags
    rs = lbm::RS_GENERAL | (wo ? lbm::RS_WOBASIS : 0) | (popbg ? lbm::RS_POPBG : 0);
  const Ops *ops = find_ops(stencil, D.precision, kspace, regime, rs);
  if (!ops) return fail(nullptr, LBM_EUNSUPPORTED, "no kernel instantiated for this combination");

  lbm_ctx *c = new lbm_ctx;
  c->stencil = stencil;
  c->space = collision_space;
  c->kspace = kspace;
  c->eq = equilibrium;
  c->zc = zc;
  c->regime = regime;
  c->prec = D.precision;
  c->streaming = D.streaming;
  c->ops = ops;
  c->rs = rs;
  c->q = q;
  c->d = two_d ? 2 : 3;
  c->gnx = D.nx;
  c->gny = D.ny;
  c->gnz = D.nz;
  c->rank = D.rank;
  c->nranks = D.nranks;
  c->swe_g = D.swe_g;
  c->device = D.device;
  c->multi = multi;
  c->dev_alloc = D.dev_alloc;
  c->dev_free = D.dev_free;
  c->alloc_user = D.alloc_user;
  c->esize = (D.precision == LBM_FP64) ? 8 : 4;
  lbm_slab_extent(slab_extent, D.rank, D.nranks, &c->offset, &c->extent);

  // memory view: (x, y, slab); D2Q9 maps its physical y onto the slab axis
  GridParams &g = c->g;
  g.nx = D.nx;
  g.ny = two_d ? 1 : D.ny;
  g.nzl = c->extent;
  g.nzg = slab_extent;
  g.z0 = c->offset;
  g.zbegin = 0;
  g.wrapz = multi ? 0 : 1;
  const size_t align = 128 / c->esize;  // 128-byte aligned rows
  g.pitch = (int)(((size_t)D.nx + align - 1) / align * align);
  g.pop = (long long)g.ny * g.pitch;
  g.plane = (long long)q * g.pop;
  int mask = 0;
  auto wall = [&](int a, int s) { return D.bc[a][s] == LBM_BC_NOSLIP; };
  if (wall(0, 0)) mask |= 1;
  if (wall(0, 1)) mask |= 2;
  if (two_d) {
    if (wall(1, 0)) mask |= 16;
    if (wall(1, 1)) mask |= 32;
  } else {
    if (wall(1, 0)) mask |= 4;
    if (wall(1, 1)) mask |= 8;
    if (wall(2, 0)) mask |= 16;
    if (wall(2, 1)) mask |= 32;
  }
  g.bcmask = mask;
  c->bb = mask != 0;

  // rates (and a zero force) in the storage precision
  for (int i = 0; i < 27; ++i) c->rates_d[i] = (i < n_rates) ? relaxation_rates[i] : 0.0;
  c->ops_plain = ops;
  fill_params(c);
  {  // temporal blocking: single rank, pull, periodic (LBM_TEMPORAL_BLOCKING=0 disables)
    const char *env = getenv("LBM_TEMPORAL_BLOCKING");
    c->tb_allowed = !(env && env[0] == '0') && D.streaming == LBM_PULL && !multi && !c->bb;
  }

  auto bail = [&](lbm_status s) {
    g_create_error = c->err;
    lbm_destroy(c);
    return s;
  };
  cudaError_t e = cudaSetDevice(D.device);
  if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaSetDevice"));
  if (wo) {  // the WO-MRT basis matrices into the kernels' constant memory (reading R31)
    double L[27 * 27], Linv[27 * 27];
    if (stencil == LBM_D2Q9) wo_basis<lbm::D2Q9>(L, Linv);
    else if (stencil == LBM_D3Q19) wo_basis<lbm::D3Q19>(L, Linv);
    else wo_basis<lbm::D3Q27>(L, Linv);
    e = (cudaError_t)ops->set_wo(L, Linv);
    if (e != cudaSuccess) return bail(cuda_fail(c, e, "WO-MRT basis upload"));
  }
  if (D.stream) {
    c->stream = (cudaStream_t)D.stream;
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaStreamCreate"));
    c->own_stream = true;
  }
  c->grid_elems = (size_t)(g.nzl + 2) * (size_t)g.plane;
  {  // two-step sweeps across ranks need 8 scratch planes (LBM_PEER_TB=0 disables, at create)
    const char *env = getenv("LBM_PEER_TB");
    c->peer_tb_cap = !(env && env[0] == '0') && multi && D.streaming == LBM_PULL && !c->bb && ops->pull2 &&
                     ops->tile_x > 0 && g.nx % ops->tile_x == 0 && g.ny % ops->tile_y == 0 && g.nzl >= 6;
    // enough CTAs for the interior sweep of one rank: >= 2 waves (the single-rank rule is 4;
    // a slab of a decomposition keeps its pairs down to 2, e.g. 8192^2 SWE on 8 ranks)
    if (c->peer_tb_cap && !(env && env[0] == '1') && tb_tiles(c) * peer_tb_chunks(c) < kTbMinCtas / 2)
      c->peer_tb_cap = false;
    c->scratch_off = c->grid_elems;
  }
  // scratch planes behind grid 0: 8 for pairs of steps across ranks, 22 more (planes 8..29) for
  // the triples of 2D contexts on the peer path (use_peer_tb3)
  const size_t alloc_elems = c->grid_elems + (c->peer_tb_cap ? (size_t)(two_d ? 30 : 8) * g.plane : 0);
  const int ngrids = (D.streaming == LBM_PULL) ? 2 : 1;
  for (int k = 0; k < ngrids; ++k) {
    if (c->dev_alloc) {
      c->buf[k] = c->dev_alloc(alloc_elems * c->esize, c->alloc_user);
      if (!c->buf[k]) return bail(fail(c, LBM_ENOMEM, "dev_alloc(populations) returned NULL"));
    } else {
      e = cudaMalloc(&c->buf[k], alloc_elems * c->esize);
      if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaMalloc(populations)"));
    }
    e = cudaMemsetAsync(c->buf[k], 0, alloc_elems * c->esize, c->stream);
    if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaMemset"));
  }
  e = cudaMalloc(&c->flag, sizeof(int));
  if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaMalloc(flag)"));
  e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaStreamSynchronize"));
  if (D.nccl_id) {  // in-library NCCL communicator (collective over the nranks ranks)
    const NcclApi &nc = nccl_api();
    if (!nc.ok) return bail(fail(c, LBM_ENCCL, nc.err));
    ncclUniqueId id;
    memcpy(&id, D.nccl_id, sizeof(id));
    const ncclResult_t r = nc.CommInitRank(&c->comm, D.nranks, id, D.rank);
    if (r != ncclSuccess) {
      c->comm = nullptr;
      return bail(fail(c, LBM_ENCCL, std::string("ncclCommInitRank: ") + nc.GetErrorString(r)));
    }
    e = cudaStreamCreateWithFlags(&c->s_int, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_i, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(cuda_fail(c, e, "NCCL exchange streams"));
  }
  *out = c;
  return LBM_OK;
}

lbm_status lbm_destroy(lbm_ctx *c) {
  if (!c) return LBM_EINVAL;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graphs(c);
  peer_release(c);
  if (c->s_int) cudaStreamSynchronize(c->s_int);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->ev_i) cudaEventDestroy(c->ev_i);
  if (c->s_int) cudaStreamDestroy(c->s_int);
  if (c->peer_flags) cudaFree(c->peer_flags);
  if (c->s_poll) cudaStreamDestroy(c->s_poll);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  if (c->comm) nccl_api().CommDestroy(c->comm);
  for (int k = 0; k < 2; ++k)
    if (c->buf[k]) {
      if (c->dev_free) c->dev_free(c->buf[k], c->alloc_user);
      else cudaFree(c->buf[k]);
    }
  if (c->staging) cudaFree(c->staging);
  if (c->flag) cudaFree(c->flag);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return LBM_OK;
}

lbm_status lbm_get_info(const lbm_ctx *c, lbm_info *info) {
  if (!c || !info) return LBM_EINVAL;
  info->q = c->q;
  info->d = c->d;
  info->offset = c->offset;
  info->extent = c->extent;
  info->nx = c->gnx;
  info->ny = c->gny;
  info->nz = c->gnz;
  info->pitch = (size_t)c->g.pitch;
  info->bytes_per_element = c->esize;
  info->device_bytes = c->grid_elems * c->esize * (c->streaming == LBM_PULL ? 2 : 1);
  info->steps_done = c->steps;
  info->rate_specialization = c->rs & 3;
  // multi-rank pull contexts with the pair sequence (peer path, in-library NCCL, or the
  // LBM_REGION_PAIR_* regions of an external exchange) run two steps per interior sweep
  info->temporal_blocking = (use_depth3(c) || (c->multi && tb3_cap(c)))
                                ? 3
                                : ((use_temporal_blocking(c) || (c->multi && c->peer_tb_cap)) ? 2 : 1);
  info->resident_cluster = resident_cluster(c);
  info->cuda_graph_steps = (c->nranks == 1 && !info->resident_cluster && use_graphs(c)) ? kGraphSteps : 0;
  info->peer_wait_host = c->peer_on && c->peer_host_wait;
  return LBM_OK;
}

lbm_status lbm_init_macroscopic(lbm_ctx *c, const double *rho, const double *u) {
  NvtxRange nvtx_("lbm_init_macroscopic");
  if (!c || !rho || !u) return fail(c, LBM_EINVAL, "null argument");
  LBM_CUDA(c, cudaSetDevice(c->device));
  const long long n = local_cells(c);
  // staging sized for lbm_get_macroscopic too (4 n doubles), so an init / get pair never frees and
  // re-allocates it (a 2 GB cudaFree + cudaMalloc cost C5's end-to-end run ~0.5 s)
  lbm_status s = ensure_staging(c, (size_t)n * 4 * sizeof(double));
  if (s != LBM_OK) return s;
  double *dr = static_cast<double *>(c->staging);
  double *du = dr + n;
  LBM_CUDA(c, cudaMemcpyAsync(dr, rho, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  LBM_CUDA(c, cudaMemcpyAsync(du, u, (size_t)n * c->d * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const int aa = c->streaming;  // storage pattern of the canonical state (kernels.cuh Canon)
  GridParams g = c->g;
  c->cur = 0;
  c->aa_state = 0;
  c->ops->init(grid_ptr(c, 0), g, aa, dr, du, c->swe_g, c->stream);
  s = check_launch(c, "k_init");
  if (s != LBM_OK) return s;
  c->steps = 0;
  c->needs_prime = c->multi;
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

lbm_status lbm_step(lbm_ctx *c, int n) {
  NvtxRange nvtx_("lbm_step");
  if (!c) return LBM_EINVAL;
  if (n < 0) return fail(c, LBM_EINVAL, "negative step count");
  if (c->multi) {  // collective: fused peer push, else the in-library NCCL exchange
    if (c->peer_on) return lbm_step_peer(c, n);
    if (!c->comm)
      return fail(c, LBM_EUNSUPPORTED,
                  "multi-rank context without a transport: lbm_peer_connect, create with nccl_id, or drive "
                  "lbm_step_region + lbm_get_halo with an external exchange");
    LBM_CUDA(c, cudaSetDevice(c->device));
    int cur = pull_parity(c);
    const lbm_status s = enqueue_nccl_steps(c, n, cur);
    if (c->streaming == LBM_PULL) c->cur = cur;
    else c->aa_state = cur;
    return s;
  }
  LBM_CUDA(c, cudaSetDevice(c->device));
  GridParams g = c->g;
  int t = 0;
  // small 2D lattices: all n steps in one cluster-resident launch (falls back to the plain
  // path for good if the cluster cannot be launched on this device)
  if (const int C = n > 0 ? resident_cluster(c) : 0) {
    const int dst = c->cur ^ (n & 1);
    const cudaError_t e = (cudaError_t)c->ops->resident(c->buf[c->cur], c->buf[dst], g, c->params, c->swe_g,
                                                         c->bb, n, C, c->stream);
    if (e == cudaSuccess) {
      c->cur = dst;
      c->steps += n;
      c->last_cluster = C;
      return check_launch(c, "k_resident2");
    }
    cudaGetLastError();
    c->resident_failed = true;
  }
  // small lattices are launch-bound: replay a captured CUDA graph of kGraphSteps steps
  if (use_graphs(c)) {
    lbm_status st = ensure_graphs(c);
    if (st != LBM_OK) return st;
    const int par = (c->streaming == LBM_PULL) ? c->cur : c->aa_state;
    for (; t + kGraphSteps <= n; t += kGraphSteps) {  // even step count: parity unchanged
      LBM_CUDA(c, cudaGraphLaunch(c->graph[par], c->stream));
      c->steps += kGraphSteps;
    }
  }
  if (use_temporal_blocking(c)) {  // triples (2D, k_pullD_2d), then pairs (k_pull2 / k_pull2_2d)
    if (use_depth3(c)) {
      for (; t + 3 <= n && n - t != 4; t += 3) {  // a remainder of 4: two pairs, not triple + single
        c->ops->pull3(c->buf[c->cur], c->buf[1 - c->cur], g, c->params, c->swe_g, tb3_zchunks(c), c->stream);
        c->cur ^= 1;
        c->steps += 3;
      }
    }
    for (; t + 2 <= n; t += 2) {
      c->ops->pull2(c->buf[c->cur], c->buf[1 - c->cur], g, c->params, c->swe_g, tb_zchunks(c), c->stream);
      c->cur ^= 1;
      c->steps += 2;
    }
  }
  for (; t < n; ++t) {
    if (c->streaming != LBM_PULL) {
      c->ops->aa(c->buf[0], g, c->params, c->swe_g, inplace_pattern(c), g.nzl, c->stream);
      c->aa_state ^= 1;
    } else {
      c->ops->pull(c->buf[c->cur], c->buf[1 - c->cur], g, c->params, c->swe_g, c->bb, g.nzl, c->stream);
      c->cur ^= 1;
    }
    c->steps++;
  }
  return check_launch(c, "stream_collide");
}

lbm_status lbm_step_region(lbm_ctx *c, lbm_region region, void *stream) {
  NvtxRange nvtx_("lbm_step_region");
  if (!c) return LBM_EINVAL;
  LBM_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  GridParams g = c->g;
  const int n = g.nzl;
  // launch the step's kernel on planes [z0, z0 + np)
  auto run = [&](int z0, int np) {
    g.zbegin = z0;
    if (c->streaming != LBM_PULL) {
      c->ops->aa(c->buf[0], g, c->params, c->swe_g, inplace_pattern(c), np, s);
    } else {
      c->ops->pull(c->buf[c->cur], c->buf[1 - c->cur], g, c->params, c->swe_g, c->bb, np, s);
    }
  };
  switch (region) {
    case LBM_REGION_ALL: run(0, n); break;
    case LBM_REGION_BOUNDARY:
      run(0, 1);
      run(n - 1, 1);
      break;
    case LBM_REGION_INTERIOR: run(1, n - 2); break;
    case LBM_REGION_PAIR_INTERIOR:
    case LBM_REGION_PAIR_BOUNDARY1:
    case LBM_REGION_PAIR_BOUNDARY2: {
      // two-step sweeps across ranks with an external exchange (the lbm_step_peer pair
      // sequence of DESIGN.md section 8, without the peer pushes)
      if (!c->peer_tb_cap)
        return fail(c, LBM_EUNSUPPORTED, "two-step regions need a multi-rank pull context with two-step sweeps");
      void *A = c->buf[c->cur], *B = c->buf[1 - c->cur];
      const size_t PB = (size_t)g.plane * c->esize;
      char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * c->esize;
      void *s_lo = scr, *s_hi = scr - (long long)(n - 6) * (long long)PB;
      GridParams gb = c->g;
      if (region == LBM_REGION_PAIR_INTERIOR) {
        gb.zbegin = 2;
        gb.zcount = n - 4;
        c->ops->pull2(A, B, gb, c->params, c->swe_g, peer_tb_chunks(c), s);
      } else if (region == LBM_REGION_PAIR_BOUNDARY1) {
        gb.zbegin = 0;
        c->ops->pull(A, s_lo, gb, c->params, c->swe_g, c->bb, 3, s);
        gb.zbegin = n - 3;
        c->ops->pull(A, s_hi, gb, c->params, c->swe_g, c->bb, 3, s);
      } else {
        gb.zbegin = 0;
        c->ops->pull(s_lo, B, gb, c->params, c->swe_g, c->bb, 2, s);
        gb.zbegin = n - 2;
        c->ops->pull(s_hi, B, gb, c->params, c->swe_g, c->bb, 2, s);
        c->steps++;  // the pair's first step (lbm_swap counts the second)
      }
      break;
    }
    case LBM_REGION_TRIPLE_INTERIOR:
    case LBM_REGION_TRIPLE_BOUNDARY1:
    case LBM_REGION_TRIPLE_BOUNDARY2:
    case LBM_REGION_TRIPLE_BOUNDARY3: {
      // three fused steps across ranks with an external exchange (the triple sequence of
      // enqueue_peer_steps without the peer pushes; scratch planes 8..29)
      if (!tb3_cap(c))
        return fail(c, LBM_EUNSUPPORTED, "three-step regions need a 2D multi-rank pull slab of >= 10 rows");
      void *A = c->buf[c->cur], *B = c->buf[1 - c->cur];
      const long long PB = (long long)g.plane * (long long)c->esize;
      char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * c->esize;
      void *l1b = scr + 8 * PB, *l1t = scr + (18 - (long long)n) * PB;
      void *l2b = scr + 20 * PB, *l2t = scr + (28 - (long long)n) * PB;
      GridParams gb = c->g;
      if (region == LBM_REGION_TRIPLE_INTERIOR) {
        gb.zbegin = 3;
        gb.zcount = n - 6;
        c->ops->pull3(A, B, gb, c->params, c->swe_g, peer_tb_chunks(c), s);
      } else if (region == LBM_REGION_TRIPLE_BOUNDARY1) {
        gb.zbegin = 0;
        c->ops->pull(A, l1b, gb, c->params, c->swe_g, c->bb, 5, s);
        gb.zbegin = n - 5;
        c->ops->pull(A, l1t, gb, c->params, c->swe_g, c->bb, 5, s);
      } else if (region == LBM_REGION_TRIPLE_BOUNDARY2) {
        gb.zbegin = 0;
        c->ops->pull(l1b, l2b, gb, c->params, c->swe_g, c->bb, 4, s);
        gb.zbegin = n - 4;
        c->ops->pull(l1t, l2t, gb, c->params, c->swe_g, c->bb, 4, s);
        c->steps++;  // the triple's first step
      } else {
        gb.zbegin = 0;
        c->ops->pull(l2b, B, gb, c->params, c->swe_g, c->bb, 3, s);
        gb.zbegin = n - 3;
        c->ops->pull(l2t, B, gb, c->params, c->swe_g, c->bb, 3, s);
        c->steps++;  // the second (lbm_swap counts the third)
      }
      break;
    }
    default: return fail(c, LBM_EINVAL, "unknown region");
  }
  return check_launch(c, "stream_collide(region)");
}

lbm_status lbm_swap(lbm_ctx *c) {
  if (!c) return LBM_EINVAL;
  if (c->streaming != LBM_PULL) c->aa_state ^= 1;
  else c->cur ^= 1;
  c->steps++;
  return LBM_OK;
}

lbm_status lbm_get_halo(lbm_ctx *c, int which, lbm_halo *out) {
  if (!c || !out) return LBM_EINVAL;
  if (c->streaming == LBM_ESOTERIC_PULL || c->streaming == LBM_ESOTERIC_TWIST || c->streaming == LBM_ESOTERIC_PUSH)
    return fail(c, LBM_EUNSUPPORTED, "Esoteric Pull / Push / Twist are single-rank");
  if (which == 2 && !c->peer_tb_cap)
    return fail(c, LBM_EUNSUPPORTED, "no scratch halo: the context does not run two-step sweeps across ranks");
  if ((which == 3 || which == 4) && !tb3_cap(c))
    return fail(c, LBM_EUNSUPPORTED, "no level scratch halo: the context does not run three-step sweeps across ranks");
  if (which < 0 || which > 4) return fail(c, LBM_EINVAL, "which must be 0 .. 4");
  lbm_layout lay;
  lbm_status s = lbm_grid_layout((lbm_stencil)c->stencil, (lbm_precision)c->prec, c->gnx, c->gny, c->gnz,
                                 c->nranks, &lay);
  if (s != LBM_OK) return fail(c, s, "layout");
  const size_t E = c->esize;
  size_t o[4] = {lay.send_lo, lay.send_hi, lay.recv_lo, lay.recv_hi};
  if (which == 3 || which == 4) {  // level-1 / level-2 scratch rows of the three-step regions
    char *p[4];
    halo_blocks(c, lay, which, c->cur, p);
    out->send_lo = p[0];
    out->send_hi = p[1];
    out->recv_lo = p[2];
    out->recv_hi = p[3];
    out->bytes = lay.halo_elems * E;
    return LBM_OK;
  }
  if (which == 2) {  // the scratch of the two-step regions: planes -1, 0 at scratch planes 0, 1
    // (the grid's offsets), planes nzl - 1, nzl at scratch planes 6, 7
    char *scr = static_cast<char *>(c->buf[0]) + c->scratch_off * E;
    const size_t shift = (size_t)(c->g.nzl - 6) * (size_t)c->g.plane;
    out->send_lo = scr + o[0] * E;
    out->send_hi = scr + (o[1] - shift) * E;
    out->recv_lo = scr + o[2] * E;
    out->recv_hi = scr + (o[3] - shift) * E;
    out->bytes = lay.halo_elems * E;
    return LBM_OK;
  }
  char *base = static_cast<char *>(grid_ptr(c, which));
  if (c->streaming == LBM_AA) {
    const size_t pre[4] = {lay.aa_pre_send_lo, lay.aa_pre_send_hi, lay.aa_pre_recv_lo, lay.aa_pre_recv_hi};
    const size_t post[4] = {lay.aa_post_send_lo, lay.aa_post_send_hi, lay.aa_post_recv_lo, lay.aa_post_recv_hi};
    for (int k = 0; k < 4; ++k) o[k] = (which == 0) ? pre[k] : post[k];
  }
  out->send_lo = base + o[0] * E;
  out->send_hi = base + o[1] * E;
  out->recv_lo = base + o[2] * E;
  out->recv_hi = base + o[3] * E;
  out->bytes = lay.halo_elems * E;
  return LBM_OK;
}

lbm_status lbm_sync(lbm_ctx *c) {
  if (!c) return LBM_EINVAL;
  LBM_CUDA(c, cudaSetDevice(c->device));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

// byte offset of p inside its allocation block (cuMemGetAddressRange, fetched through the runtime:
// no -lcuda); the block is what a CUDA IPC handle of p names
static lbm_status allocation_offset(lbm_ctx *c, void *p, long long *off) {
  typedef CUresult (*RangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);
  static RangeFn range = nullptr;
  if (!range) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    const cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess)
      return fail(c, LBM_ECUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<RangeFn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    return fail(c, LBM_ECUDA, "cuMemGetAddressRange failed");
  *off = (long long)(reinterpret_cast<CUdeviceptr>(p) - base);
  return LBM_OK;
}

lbm_status lbm_peer_export(lbm_ctx *c, lbm_peer_info *out) {
  if (!c || !out) return LBM_EINVAL;
  if (c->streaming == LBM_ESOTERIC_PULL || c->streaming == LBM_ESOTERIC_TWIST || c->streaming == LBM_ESOTERIC_PUSH)
    return fail(c, LBM_EUNSUPPORTED, "Esoteric Pull / Push / Twist are single-rank");
  if (c->nranks < 2) return fail(c, LBM_EUNSUPPORTED, "the fused halo push needs nranks > 1");
  LBM_CUDA(c, cudaSetDevice(c->device));
  if (!c->peer_flags) {
    LBM_CUDA(c, cudaMalloc(&c->peer_flags, 4 * sizeof(long long)));
    LBM_CUDA(c, cudaMemset(c->peer_flags, 0, 4 * sizeof(long long)));
  }
  memset(out, 0, sizeof(*out));
  for (int k = 0; k < 2; ++k) {
    if (!c->buf[k]) continue;  // in place (AA): one grid
    cudaIpcMemHandle_t h;
    LBM_CUDA(c, cudaIpcGetMemHandle(&h, c->buf[k]));
    memcpy(out->grid_ipc[k], &h, sizeof(h));
    out->grid[k] = c->buf[k];
    // the handle names the whole allocation block: a grid sub-allocated through dev_alloc (a
    // caching allocator) sits at an offset inside it, which the importer adds back
    out->grid_off[k] = 0;
    if (c->dev_alloc) {
      long long off = 0;
      if (lbm_status s = allocation_offset(c, c->buf[k], &off); s != LBM_OK) return s;
      out->grid_off[k] = off;
    }
  }
  cudaIpcMemHandle_t h;
  LBM_CUDA(c, cudaIpcGetMemHandle(&h, c->peer_flags));
  memcpy(out->flags_ipc, &h, sizeof(h));
  out->flags = c->peer_flags;
  out->pid = (long long)getpid();
  out->device = c->device;
  out->rank = c->rank;
  out->nranks = c->nranks;
  out->stencil = c->stencil;
  out->precision = c->prec;
  out->nx = c->gnx;
  out->ny = c->gny;
  out->nz = c->gnz;
  cudaDeviceProp prop{};
  LBM_CUDA(c, cudaGetDeviceProperties(&prop, c->device));
  memcpy(out->uuid, &prop.uuid, sizeof(out->uuid));
  memcpy(c->uuid, &prop.uuid, sizeof(c->uuid));
  return LBM_OK;
}

lbm_status peer_connect_impl(lbm_ctx *c, const lbm_peer_info *lo, const lbm_peer_info *hi);

lbm_status lbm_peer_connect(lbm_ctx *c, const lbm_peer_info *lo, const lbm_peer_info *hi) {
  NvtxRange nvtx_("lbm_peer_connect");
  if (!c || (!lo) != (!hi)) return LBM_EINVAL;
  if (!lo) {  // disconnect: unmap the neighbours (back to lbm_step_region + an external exchange)
    LBM_CUDA(c, cudaSetDevice(c->device));
    LBM_CUDA(c, cudaDeviceSynchronize());
    peer_release(c);
    drop_graphs(c);
    return LBM_OK;
  }
  const lbm_status s = peer_connect_impl(c, lo, hi);
  if (s != LBM_OK) peer_release(c);  // no half-mapped ring stays behind
  return s;
}

lbm_status peer_connect_impl(lbm_ctx *c, const lbm_peer_info *lo, const lbm_peer_info *hi) {
  if (!c->peer_flags) return fail(c, LBM_EINVAL, "lbm_peer_export first");
  const lbm_peer_info *nb[2] = {lo, hi};
  const int want[2] = {(c->rank + c->nranks - 1) % c->nranks, (c->rank + 1) % c->nranks};
  for (int k = 0; k < 2; ++k) {
    const lbm_peer_info *p = nb[k];
    if (p->nranks != c->nranks || p->rank != want[k] || p->stencil != c->stencil || p->precision != c->prec ||
        p->nx != c->gnx || p->ny != c->gny || p->nz != c->gnz)
      return fail(c, LBM_EINVAL, "peer info does not match this context's slab ring");
  }
  LBM_CUDA(c, cudaSetDevice(c->device));
  LBM_CUDA(c, cudaDeviceSynchronize());
  peer_release(c);
  drop_graphs(c);  // captured peer loops hold the old neighbour pointers
  const long long me = (long long)getpid();
  // maps a peer allocation: same process -> its pointer; else CUDA IPC (one mapping per handle)
  auto map = [&](const lbm_peer_info *p, const unsigned char *ipc, void *raw, long long off, void **out) -> lbm_status {
    if (p->pid == me) {
      if (p->device != c->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(p->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return cuda_fail(c, e, "cudaDeviceEnablePeerAccess");
      }
      *out = raw;
      return LBM_OK;
    }
    for (int k = 0; k < c->n_mapped; ++k)  // the same neighbour on both sides (two ranks)
      if (c->peer_pid[k] == p->pid && c->peer_raw[k] == raw) {
        *out = static_cast<char *>(c->peer_mapped[k]) + off;
        return LBM_OK;
      }
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc, sizeof(h));
    void *ptr = nullptr;
    LBM_CUDA(c, cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer_pid[c->n_mapped] = p->pid;
    c->peer_raw[c->n_mapped] = raw;
    c->peer_mapped[c->n_mapped++] = ptr;  // the block base (what cudaIpcCloseMemHandle takes)
    *out = static_cast<char *>(ptr) + off;
    return LBM_OK;
  };
  void *g[2][2], *f[2];
  for (int k = 0; k < 2; ++k) {
    const lbm_peer_info *p = nb[k];
    lbm_status s;
    if ((s = map(p, p->grid_ipc[0], p->grid[0], p->grid_off[0], &g[0][k])) != LBM_OK) return s;
    g[1][k] = nullptr;
    if (p->grid[1] && (s = map(p, p->grid_ipc[1], p->grid[1], p->grid_off[1], &g[1][k])) != LBM_OK) return s;
    if ((s = map(p, p->flags_ipc, p->flags, 0, &f[k])) != LBM_OK) return s;
  }
  const size_t P = c->g.plane * c->esize, nzl = (size_t)c->g.nzl;
  for (int b = 0; b < 2; ++b) {
    for (int k = 0; k < 2; ++k) c->peer_base[b][k] = g[b][k];
    if (c->streaming == LBM_PULL) {
      c->peer_ghost[b][0] = static_cast<char *>(g[b][0]) + (nzl + 1) * P;  // lower's top ghost plane
      c->peer_ghost[b][1] = g[b][1];                                        // upper's bottom ghost plane
    } else if (b == 0) {
      c->peer_ghost[0][0] = static_cast<char *>(g[0][0]) + nzl * P;  // AA: lower's last plane
      c->peer_ghost[0][1] = static_cast<char *>(g[0][1]) + P;        // AA: upper's first plane
    }
  }
  for (int k = 0; k < 2; ++k)  // the neighbours' scratch planes (two-step sweeps across ranks)
    c->peer_scr[k] = c->peer_tb_cap ? static_cast<char *>(g[0][k]) + c->scratch_off * c->esize : nullptr;
  c->peer_remote[0] = static_cast<long long *>(f[0]) + 1;  // I am the lower's upper neighbour
  c->peer_remote[1] = static_cast<long long *>(f[1]) + 0;
  LBM_CUDA(c, cudaMemset(c->peer_flags, 0, 4 * sizeof(long long)));
  // device-side waits only when every neighbour runs on another GPU (peer_wait)
  {
    bool shared = false;
    for (int k = 0; k < 2; ++k) shared |= memcmp(nb[k]->uuid, c->uuid, sizeof(c->uuid)) == 0;
    const char *env = getenv("LBM_PEER_WAIT");
    c->peer_host_wait = env && !strcmp(env, "host") ? true : env && !strcmp(env, "device") ? false : shared;
    c->host_phase = 0;
    c->host_timed_out = false;
    if (c->peer_host_wait && !c->s_poll) {
      LBM_CUDA(c, cudaStreamCreateWithFlags(&c->s_poll, cudaStreamNonBlocking));
      LBM_CUDA(c, cudaMallocHost(&c->h_flags, 2 * sizeof(long long)));
    }
  }
  // load the wait / signal kernels and every step kernel now, before any wait can spin
  // (lazy module loading at a first launch waits for the running kernels: Ops::preload)
  {
    cudaFuncAttributes a{};
    LBM_CUDA(c, cudaFuncGetAttributes(&a, k_peer_wait));
    LBM_CUDA(c, cudaFuncGetAttributes(&a, k_peer_signal));
    c->ops->preload();
    if (c->ops_plain != c->ops) c->ops_plain->preload();
  }
  if (!c->s_int) {
    LBM_CUDA(c, cudaStreamCreateWithFlags(&c->s_int, cudaStreamNonBlocking));
    LBM_CUDA(c, cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming));
    LBM_CUDA(c, cudaEventCreateWithFlags(&c->ev_i, cudaEventDisableTiming));
  }
  LBM_CUDA(c, cudaDeviceSynchronize());
  c->peer_on = true;
  return LBM_OK;
}

lbm_status lbm_peer_prime(lbm_ctx *c) {
  NvtxRange nvtx_("lbm_peer_prime");
  if (!c) return LBM_EINVAL;
  if (!c->peer_on) return fail(c, LBM_EINVAL, "lbm_peer_connect first");
  LBM_CUDA(c, cudaSetDevice(c->device));
  c->needs_prime = false;
  lbm_layout lay;
  lbm_status s = lbm_grid_layout((lbm_stencil)c->stencil, (lbm_precision)c->prec, c->gnx, c->gny, c->gnz,
                                 c->nranks, &lay);
  if (s != LBM_OK) return fail(c, s, "layout");
  const size_t E = c->esize, bytes = lay.halo_elems * E;
  if (c->streaming != LBM_PULL) {  // AA: no ghost data; the handshake orders the neighbours' init
    peer_wait(c, peer_timeout_ns());
    peer_signal(c);
    return check_launch(c, "lbm_peer_prime");
  }
  const int b = c->cur;
  const char *base = static_cast<const char *>(c->buf[b]);
  const size_t top = (size_t)(c->g.nzl + 1) * c->g.plane * E;
  // the ghost plane offsets of the receive blocks (recv_hi lies in plane nzl + 1, recv_lo in 0)
  char *lo_dst = static_cast<char *>(c->peer_ghost[b][0]) - top + lay.recv_hi * E;
  char *hi_dst = static_cast<char *>(c->peer_ghost[b][1]) + lay.recv_lo * E;
  peer_wait(c, peer_timeout_ns());
  LBM_CUDA(c, cudaMemcpyAsync(lo_dst, base + lay.send_lo * E, bytes, cudaMemcpyDefault, c->stream));
  LBM_CUDA(c, cudaMemcpyAsync(hi_dst, base + lay.send_hi * E, bytes, cudaMemcpyDefault, c->stream));
  peer_signal(c);
  return check_launch(c, "lbm_peer_prime");
}

lbm_status lbm_step_peer(lbm_ctx *c, int n) {
  NvtxRange nvtx_("lbm_step_peer");
  if (!c) return LBM_EINVAL;
  if (n < 0) return fail(c, LBM_EINVAL, "negative step count");
  if (!c->peer_on) return fail(c, LBM_EINVAL, "lbm_peer_connect first");
  LBM_CUDA(c, cudaSetDevice(c->device));
  if (c->needs_prime) {  // after init / set: push the current boundary planes first
    const lbm_status ps = lbm_peer_prime(c);
    if (ps != LBM_OK) return ps;
  }
  int t = 0;
  // steps per captured loop: an even number of grid swaps (32 single steps or pairs; 36 = 12
  // triples on the 2D peer path), so a graph ends on the parity it started from
  const int gsteps = use_peer_tb3(c) ? 36 : kGraphSteps;
  if ((c->peer_graph[0] || c->peer_graph[1]) && c->peer_graph_steps != gsteps) drop_graphs(c);
  if (n >= gsteps && graphs_enabled() && !c->peer_host_wait) {  // replay captured step loops
    c->peer_graph_steps = gsteps;
    for (int par = 0; par < 2; ++par) {
      if (c->peer_graph[par]) continue;
      cudaGraph_t gr = nullptr;
      LBM_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      const int endp = enqueue_peer_steps(c, gsteps, par);  // par: pull grid / AA state
      cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
      if (e == cudaSuccess && endp != par) e = cudaErrorInvalidValue;  // odd number of swaps
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaGraphInstantiate(&c->peer_graph[par], gr, 0);
      if (gr) cudaGraphDestroy(gr);
      if (e != cudaSuccess) {
        c->peer_graph[par] = nullptr;
        return cuda_fail(c, e, "CUDA-graph capture of the peer step loop");
      }
    }
    const int par = pull_parity(c);
    for (; t + gsteps <= n; t += gsteps) {  // an even number of swaps: the parity is unchanged
      LBM_CUDA(c, cudaGraphLaunch(c->peer_graph[par], c->stream));
      c->steps += gsteps;
    }
  }
  if (t < n) {
    const int end = enqueue_peer_steps(c, n - t, pull_parity(c));
    if (c->streaming == LBM_PULL) c->cur = end;
    else c->aa_state = end;
    c->steps += n - t;
  }
  return check_launch(c, "lbm_step_peer");
}

lbm_status lbm_peer_status(lbm_ctx *c, int *timed_out) {
  if (!c || !timed_out) return LBM_EINVAL;
  if (!c->peer_flags) {
    *timed_out = 0;
    return LBM_OK;
  }
  LBM_CUDA(c, cudaSetDevice(c->device));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  long long v = 0;
  LBM_CUDA(c, cudaMemcpy(&v, c->peer_flags + 2, sizeof(v), cudaMemcpyDeviceToHost));
  *timed_out = v != 0 || c->host_timed_out;
  return LBM_OK;
}

lbm_status lbm_get_macroscopic(lbm_ctx *c, double *rho, double *u) {
  NvtxRange nvtx_("lbm_get_macroscopic");
  if (!c || !rho || !u) return fail(c, LBM_EINVAL, "null argument");
  LBM_CUDA(c, cudaSetDevice(c->device));
  if (lbm_status ps = peer_refresh(c); ps != LBM_OK) return ps;
  const long long n = local_cells(c);
  lbm_status s = ensure_staging(c, (size_t)n * 4 * sizeof(double));
  if (s != LBM_OK) return s;
  double *dr = static_cast<double *>(c->staging);
  double *du = dr + n;
  const int aa = c->streaming;  // storage pattern of the canonical state (kernels.cuh Canon)
  c->ops->macro(grid_ptr(c, 0), c->g, aa, c->aa_state, c->zc, dr, du, post_shift(c), c->stream);
  s = check_launch(c, "k_macroscopic");
  if (s != LBM_OK) return s;
  LBM_CUDA(c, cudaMemcpyAsync(rho, dr, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaMemcpyAsync(u, du, (size_t)n * c->d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

lbm_status lbm_get_populations(lbm_ctx *c, double *f) {
  NvtxRange nvtx_("lbm_get_populations");
  if (!c || !f) return fail(c, LBM_EINVAL, "null argument");
  LBM_CUDA(c, cudaSetDevice(c->device));
  if (lbm_status ps = peer_refresh(c); ps != LBM_OK) return ps;
  const long long n = local_cells(c);
  const size_t bytes = (size_t)n * c->q * sizeof(double);
  lbm_status s = ensure_staging(c, bytes);
  if (s != LBM_OK) return s;
  const int aa = c->streaming;  // storage pattern of the canonical state (kernels.cuh Canon)
  c->ops->get_pop(grid_ptr(c, 0), c->g, aa, c->aa_state, static_cast<double *>(c->staging), c->stream);
  s = check_launch(c, "k_get_populations");
  if (s != LBM_OK) return s;
  LBM_CUDA(c, cudaMemcpyAsync(f, c->staging, bytes, cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

lbm_status lbm_set_force(lbm_ctx *c, const double *force) {
  if (!c || !force) return fail(c, LBM_EINVAL, "null argument");
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(force[a])) return fail(c, LBM_EINVAL, "non-finite force");
  if (c->d == 2 && force[2] != 0.0) return fail(c, LBM_EINVAL, "a D2Q9 force has no z component");
  const bool any = force[0] != 0.0 || force[1] != 0.0 || force[2] != 0.0;
  if (any) {
    if (c->rs & lbm::RS_DISCRETE)
      return fail(c, LBM_EUNSUPPORTED, "no body force with the discrete equilibrium (reading R29)");
    if (c->rs & (lbm::RS_WOBASIS | lbm::RS_POPBG))
      return fail(c, LBM_EUNSUPPORTED, "no body force with the WO-MRT basis or LBM_EQ_ABSOLUTE_F0");
    if (!(c->kspace == LBM_SPACE_POPULATION || c->kspace == LBM_SPACE_RAW || c->kspace == LBM_SPACE_CENTRAL ||
          c->kspace == LBM_SPACE_CUMULANT))
      return fail(c, LBM_EUNSUPPORTED,
                  "a body force is provided for population, raw-moment, central-moment and cumulant collisions "
                  "(readings R23, R26), not for shallow water");
    // He and Guo coincide for the cumulant methods (readings R26, R27): one kernel
    const bool he = c->force_model == LBM_FORCE_HE && c->kspace != LBM_SPACE_CUMULANT;
    const Ops *f = find_ops(c->stencil, c->prec, c->kspace, c->regime,
                            lbm::RS_GENERAL | (he ? lbm::RS_FORCE_HE : lbm::RS_FORCE));
    if (!f) return fail(c, LBM_EUNSUPPORTED, "no forced kernel instantiated for this combination");
    c->ops = f;
    if (c->peer_on) f->preload();  // before any neighbour wait can spin (Ops::preload)
  } else {
    c->ops = c->ops_plain;
  }
  for (int a = 0; a < 3; ++a) c->force[a] = force[a];
  c->forced = any;
  fill_params(c);
  drop_graphs(c);  // the captured launches hold the old parameters by value
  return LBM_OK;
}

lbm_status lbm_set_force_model(lbm_ctx *c, lbm_force_model model) {
  if (!c) return fail(c, LBM_EINVAL, "null argument");
  if (model != LBM_FORCE_GUO && model != LBM_FORCE_HE) return fail(c, LBM_EINVAL, "unknown force model");
  const int old = c->force_model;
  c->force_model = model;
  if (!c->forced) return LBM_OK;
  const lbm_status s = lbm_set_force(c, c->force);  // re-selects the forced kernels
  if (s != LBM_OK) c->force_model = old;
  return s;
}

lbm_status lbm_get_diagnostics(lbm_ctx *c, lbm_diagnostics *out) {
  NvtxRange nvtx_("lbm_get_diagnostics");
  if (!c || !out) return fail(c, LBM_EINVAL, "null argument");
  LBM_CUDA(c, cudaSetDevice(c->device));
  if (lbm_status ps = peer_refresh(c); ps != LBM_OK) return ps;
  const size_t pbytes = (size_t)5 * lbm::DIAG_GRID * sizeof(double);
  lbm_status s = ensure_staging(c, pbytes + 5 * sizeof(double));
  if (s != LBM_OK) return s;
  double *partial = static_cast<double *>(c->staging);
  double *dout = partial + 5 * lbm::DIAG_GRID;
  c->ops->diagnostics(grid_ptr(c, 0), c->g, c->streaming, c->aa_state, c->zc, partial, dout,
                      post_shift(c), c->stream);
  s = check_launch(c, "k_diag");
  if (s != LBM_OK) return s;
  double h[5];
  LBM_CUDA(c, cudaMemcpyAsync(h, dout, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  out->mass = h[0];
  out->momentum[0] = h[1];
  out->momentum[1] = h[2];
  out->momentum[2] = h[3];
  out->kinetic_energy = h[4];
  return LBM_OK;
}

lbm_status lbm_get_cells(lbm_ctx *c, const long long *cells, long long n, double *f) {
  if (!c || (n > 0 && (!cells || !f)) || n < 0) return fail(c, LBM_EINVAL, "bad argument");
  if (n == 0) return LBM_OK;
  const long long ncell = local_cells(c);
  for (long long k = 0; k < n; ++k)
    if (cells[k] < 0 || cells[k] >= ncell) return fail(c, LBM_EINVAL, "cell index out of range");
  LBM_CUDA(c, cudaSetDevice(c->device));
  if (lbm_status ps = peer_refresh(c); ps != LBM_OK) return ps;
  const size_t ibytes = (size_t)n * sizeof(long long), obytes = (size_t)n * c->q * sizeof(double);
  lbm_status s = ensure_staging(c, ibytes + obytes + 256);
  if (s != LBM_OK) return s;
  long long *didx = static_cast<long long *>(c->staging);
  double *dout = reinterpret_cast<double *>(static_cast<char *>(c->staging) + (ibytes + 255) / 256 * 256);
  LBM_CUDA(c, cudaMemcpyAsync(didx, cells, ibytes, cudaMemcpyHostToDevice, c->stream));
  c->ops->get_cells(grid_ptr(c, 0), c->g, c->streaming, c->aa_state, didx, n, dout, c->stream);
  s = check_launch(c, "k_get_cells");
  if (s != LBM_OK) return s;
  LBM_CUDA(c, cudaMemcpyAsync(f, dout, obytes, cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

lbm_status lbm_set_steps(lbm_ctx *c, long long steps) {
  if (!c) return LBM_EINVAL;
  if (steps < 0) return fail(c, LBM_EINVAL, "negative step count");
  c->steps = steps;
  return LBM_OK;
}

lbm_status lbm_set_populations(lbm_ctx *c, const double *f) {
  NvtxRange nvtx_("lbm_set_populations");
  if (!c || !f) return fail(c, LBM_EINVAL, "null argument");
  LBM_CUDA(c, cudaSetDevice(c->device));
  const long long n = local_cells(c);
  const size_t bytes = (size_t)n * c->q * sizeof(double);
  lbm_status s = ensure_staging(c, bytes);
  if (s != LBM_OK) return s;
  LBM_CUDA(c, cudaMemcpyAsync(c->staging, f, bytes, cudaMemcpyHostToDevice, c->stream));
  const int aa = c->streaming;  // storage pattern of the canonical state (kernels.cuh Canon)
  c->cur = 0;
  c->aa_state = 0;
  c->ops->set_pop(grid_ptr(c, 0), c->g, aa, static_cast<const double *>(c->staging), c->stream);
  s = check_launch(c, "k_set_populations");
  if (s != LBM_OK) return s;
  c->steps = 0;
  c->needs_prime = c->multi;
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

lbm_status lbm_check_finite(lbm_ctx *c) {
  if (!c) return LBM_EINVAL;
  LBM_CUDA(c, cudaSetDevice(c->device));
  LBM_CUDA(c, cudaMemsetAsync(c->flag, 0, sizeof(int), c->stream));
  c->ops->check_finite(grid_ptr(c, 0), c->g, c->flag, c->stream);
  lbm_status s = check_launch(c, "k_check_finite");
  if (s != LBM_OK) return s;
  int h = 0;
  LBM_CUDA(c, cudaMemcpyAsync(&h, c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  if (h) return fail(c, LBM_ENUMERIC, "non-finite population after step " + std::to_string(c->steps));
  return LBM_OK;
}

lbm_status lbm_test_collide(lbm_ctx *c, const double *f_in, double *f_out, long long n_cells) {
  if (!c || !f_in || !f_out || n_cells < 0) return fail(c, LBM_EINVAL, "bad argument");
  if (n_cells == 0) return LBM_OK;
  LBM_CUDA(c, cudaSetDevice(c->device));
  const size_t bytes = (size_t)n_cells * c->q * sizeof(double);
  lbm_status s = ensure_staging(c, 2 * bytes);
  if (s != LBM_OK) return s;
  double *din = static_cast<double *>(c->staging);
  double *dout = din + (size_t)n_cells * c->q;
  LBM_CUDA(c, cudaMemcpyAsync(din, f_in, bytes, cudaMemcpyHostToDevice, c->stream));
  c->ops->test_collide(din, dout, n_cells, c->params, c->swe_g, c->stream);
  s = check_launch(c, "k_test_collide");
  if (s != LBM_OK) return s;
  LBM_CUDA(c, cudaMemcpyAsync(f_out, dout, bytes, cudaMemcpyDeviceToHost, c->stream));
  LBM_CUDA(c, cudaStreamSynchronize(c->stream));
  return LBM_OK;
}

/* diagnostics: registers / local memory of the kernel that dominates this context's lbm_step */
lbm_status lbm_kernel_attributes(const lbm_ctx *c, int *regs, int *local_bytes) {
  if (!c || !regs || !local_bytes) return LBM_EINVAL;
  int which = 0;
  if (resident_cluster(c)) which = 2;
  else if (use_depth3(c)) which = 3;
  else if (use_temporal_blocking(c) || (c->multi && c->peer_tb_cap)) which = 1;
  else if (c->streaming != LBM_PULL) which = 10 + inplace_pattern(c, 0);
  c->ops->attributes(which, regs, local_bytes);
  return LBM_OK;
}

/* device pointer of the current population grid (for zero-copy diagnostics) */
lbm_status lbm_device_grid(lbm_ctx *c, int which, void **ptr, size_t *bytes) {
  if (!c || !ptr || !bytes) return LBM_EINVAL;
  *ptr = grid_ptr(c, which);
  *bytes = c->grid_elems * c->esize;
  return LBM_OK;
}

/* the context's CUDA stream (cudaStream_t) */
void *lbm_stream(lbm_ctx *c) { return c ? (void *)c->stream : nullptr; }

}  // extern "C"
