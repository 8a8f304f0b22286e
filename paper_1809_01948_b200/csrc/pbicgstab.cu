// pbicgstab.cu -- host driver and C ABI (include/pbicgstab.h) of the B200
// p-BiCGStab library.  One translation unit, compiled with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
// (no FMA contraction anywhere: reading A4).
//
// Host responsibilities only: validation, workspace allocation, launch order,
// CUDA-graph capture/replay of chunks of iterations, asynchronous polling of the
// device `done` flag, history download.  Every arithmetic step of Alg. 2 runs in
// the kernels of stencil_kernels.cuh / csr_kernels.cuh.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/pbicgstab.h"
#include "csr_kernels.cuh"
#include "stencil_kernels.cuh"
#include "tile_sweeps.cuh"

namespace {

thread_local std::string g_create_err;

enum Kname { K_INIT = 0, K_SWEEPA, K_SWEEPC, K_SPMVB, K_SPMVD, K_RR1, K_RR2, K_GAP, K_APPLY, K_N };
const char* kname_str[K_N] = {"init", "sweepA", "sweepC", "spmvB", "spmvD",
                              "rr1",  "rr2",    "gap",    "apply"};

struct TimedLaunch {
  int k;
  cudaEvent_t e0, e1;
};

enum Kind { KIND_STENCIL = 0, KIND_CSR = 1 };

}  // namespace

struct pbicg_ctx {
  int kind = KIND_STENCIL;
  int dim = 3;
  int device = 0, num_sm = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_entry = nullptr, ev_poll[2] = {nullptr, nullptr};
  int64_t n_local = 0, row_begin = 0, n_global = 0, H = 0;
  Geo geo{};
  TileGeo tg{};
  bool tile_ok = false;  // TMA 2.5D sweeps eligible for this operator
  int tile_on = 1;       // option "tile"
  size_t tile_smem[2] = {0, 0};
  CsrOp csr{};
  std::vector<void*> allocs;
  Vecs V{};
  double* xtmp = nullptr;  // ghosted scratch for pbicgstab_apply
  Scal* scal = nullptr;
  Scal* scal_host = nullptr;  // pinned, [2] (poll double buffer)
  Dd* part = nullptr;
  Hist hist{nullptr, nullptr};
  int64_t hist_cap = 0;
  int block = 256;
  int grid[K_N] = {0};
  // options
  int bench = 0, use_graphs = 1, timing = 0, overlap = 1, schedule = 0, gap_on = 0;
  int rr_period_cur = 0;
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs;
  std::vector<TimedLaunch> pending;
  std::vector<cudaEvent_t> ev_pool;
  int64_t launches[K_N] = {0};
  double ms[K_N] = {0};
  bool failed = false;
  std::string err;
};

namespace {

pbicg_status fail(pbicg_ctx* h, pbicg_status st, const std::string& msg) {
  if (h) {
    h->err = msg;
  } else {
    g_create_err = msg;
  }
  return st;
}

#define CU(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      return fail(h, PBICG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                                    \
  } while (0)

pbicg_status dalloc(pbicg_ctx* h, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 8);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, PBICG_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) +
                                     "): " + cudaGetErrorString(e));
  }
  h->allocs.push_back(*p);
  return PBICG_OK;
}

// ghosted vector: H doubles before and after n_local rows, zero-filled
pbicg_status gvec(pbicg_ctx* h, double** out) {
  void* p = nullptr;
  size_t n = (size_t)(h->n_local + 2 * h->H);
  pbicg_status st = dalloc(h, &p, n * sizeof(double));
  if (st) return st;
  CU(cudaMemsetAsync(p, 0, n * sizeof(double), h->stream));
  *out = (double*)p + h->H;
  return PBICG_OK;
}

template <typename KernelT>
int occ_grid(pbicg_ctx* h, KernelT kern, int64_t work_items) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, h->block, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t g = (int64_t)per_sm * h->num_sm;
  if (g > work_items) g = work_items;
  if (g < 1) g = 1;
  return (int)g;
}

cudaEvent_t pool_event(pbicg_ctx* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Launch bookkeeping: counts every launch, brackets it with events in timing mode.
struct LaunchScope {
  pbicg_ctx* h;
  int k;
  cudaEvent_t e0 = nullptr;
  LaunchScope(pbicg_ctx* h_, int k_) : h(h_), k(k_) {
    h->launches[k]++;
    if (h->timing) {
      e0 = pool_event(h);
      cudaEventRecord(e0, h->stream);
    }
  }
  ~LaunchScope() {
    if (h->timing) {
      cudaEvent_t e1 = pool_event(h);
      cudaEventRecord(e1, h->stream);
      h->pending.push_back({k, e0, e1});
    }
  }
};

void collect_timing(pbicg_ctx* h) {
  for (auto& t : h->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.e0, t.e1) == cudaSuccess) h->ms[t.k] += ms;
    h->ev_pool.push_back(t.e0);
    h->ev_pool.push_back(t.e1);
  }
  h->pending.clear();
  cudaGetLastError();
}

// ---------------------------------------------------------------------------
// enqueue helpers (stencil, fused 2-sweep schedule; CSR, split 4-phase)
template <int DIM>
void enq_init_stencil(pbicg_ctx* h) {
  { LaunchScope ls(h, K_INIT);
    k_init1<DIM><<<h->grid[K_INIT], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part); }
  { LaunchScope ls(h, K_INIT);
    k_init2<DIM><<<h->grid[K_INIT], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part,
                                                                h->hist); }
}

template <int DIM>
void enq_iter_stencil(pbicg_ctx* h, bool with_rr, bool with_gap) {
  if (h->tile_ok && h->tile_on) {
    { LaunchScope ls(h, K_SWEEPA);
      t_sweep<DIM, 0><<<h->tg.units < h->num_sm ? h->tg.units : h->num_sm, TNT, h->tile_smem[0],
                         h->stream>>>(h->tg, h->V, h->scal, h->part, h->hist); }
    { LaunchScope ls(h, K_SWEEPC);
      t_sweep<DIM, 1><<<h->tg.units < h->num_sm ? h->tg.units : h->num_sm, TNT, h->tile_smem[1],
                         h->stream>>>(h->tg, h->V, h->scal, h->part, h->hist); }
  } else {
    { LaunchScope ls(h, K_SWEEPA);
      k_sweepA<DIM><<<h->grid[K_SWEEPA], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part); }
    { LaunchScope ls(h, K_SWEEPC);
      k_sweepC<DIM><<<h->grid[K_SWEEPC], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part,
                                                                     h->hist); }
  }
  if (with_rr) {
    { LaunchScope ls(h, K_RR1);
      k_rr1<DIM><<<h->grid[K_RR1], h->block, 0, h->stream>>>(h->geo, h->V, h->scal); }
    { LaunchScope ls(h, K_RR2);
      k_rr2<DIM><<<h->grid[K_RR2], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part,
                                                               h->hist); }
  }
  if (with_gap) {
    LaunchScope ls(h, K_GAP);
    k_gap<DIM><<<h->grid[K_GAP], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part,
                                                             h->hist);
  }
}

void enq_gap(pbicg_ctx* h) {
  if (h->kind == KIND_CSR) {
    LaunchScope ls(h, K_GAP);
    c_gap<<<h->grid[K_GAP], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part, h->hist);
  } else if (h->dim == 3) {
    LaunchScope ls(h, K_GAP);
    k_gap<3><<<h->grid[K_GAP], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part, h->hist);
  } else {
    LaunchScope ls(h, K_GAP);
    k_gap<2><<<h->grid[K_GAP], h->block, 0, h->stream>>>(h->geo, h->V, h->scal, h->part, h->hist);
  }
}

void enq_init_csr(pbicg_ctx* h) {
  { LaunchScope ls(h, K_INIT);
    c_init1<<<h->grid[K_INIT], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part); }
  { LaunchScope ls(h, K_INIT);
    c_init2<<<h->grid[K_INIT], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part, h->hist); }
  { LaunchScope ls(h, K_SPMVD);  // t_0 = A m_0 (line 3)
    c_spmvD<<<h->grid[K_SPMVD], h->block, 0, h->stream>>>(h->csr, h->V, h->scal); }
}

void enq_iter_csr(pbicg_ctx* h, bool with_rr, bool with_gap) {
  { LaunchScope ls(h, K_SWEEPA);
    c_sweepA<<<h->grid[K_SWEEPA], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part); }
  { LaunchScope ls(h, K_SPMVB);
    c_spmvB<<<h->grid[K_SPMVB], h->block, 0, h->stream>>>(h->csr, h->V, h->scal); }
  { LaunchScope ls(h, K_SWEEPC);
    c_sweepC<<<h->grid[K_SWEEPC], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part, h->hist); }
  if (with_rr) {
    { LaunchScope ls(h, K_RR1);
      c_rr1<<<h->grid[K_RR1], h->block, 0, h->stream>>>(h->csr, h->V, h->scal); }
    { LaunchScope ls(h, K_RR2);
      c_rr2<<<h->grid[K_RR2], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part, h->hist); }
  }
  { LaunchScope ls(h, K_SPMVD);
    c_spmvD<<<h->grid[K_SPMVD], h->block, 0, h->stream>>>(h->csr, h->V, h->scal); }
  if (with_gap) enq_gap(h);
}

void enq_init(pbicg_ctx* h) {
  if (h->kind == KIND_CSR) enq_init_csr(h);
  else if (h->dim == 3) enq_init_stencil<3>(h);
  else enq_init_stencil<2>(h);
  if (h->gap_on) enq_gap(h);
}

void enq_iter(pbicg_ctx* h, bool with_rr) {
  if (h->kind == KIND_CSR) enq_iter_csr(h, with_rr, h->gap_on);
  else if (h->dim == 3) enq_iter_stencil<3>(h, with_rr, h->gap_on);
  else enq_iter_stencil<2>(h, with_rr, h->gap_on);
}

// chunk of L iterations starting at a multiple of L (L a multiple of P when P>0):
// iteration offset o replaces iff P > 0 && (o+1) % P == 0.
void enq_chunk(pbicg_ctx* h, int L, int P) {
  for (int o = 0; o < L; ++o) enq_iter(h, P > 0 && ((o + 1) % P) == 0);
}

pbicg_status run_chunk(pbicg_ctx* h, int L, int P) {
  if (!h->use_graphs || h->timing) {
    enq_chunk(h, L, P);
    CU(cudaGetLastError());
    return PBICG_OK;
  }
  auto key = std::make_tuple(L, P, h->gap_on);
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    // capture without counting: counts are added per replay below
    int64_t saved[K_N];
    memcpy(saved, h->launches, sizeof(saved));
    CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    enq_chunk(h, L, P);
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
    memcpy(h->launches, saved, sizeof(saved));
    if (ce != cudaSuccess) return fail(h, PBICG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t ge = nullptr;
    ce = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(h, PBICG_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    it = h->graphs.emplace(key, ge).first;
  }
  CU(cudaGraphLaunch(it->second, h->stream));
  // account the replay's launches
  for (int o = 0; o < L; ++o) {
    bool rr = P > 0 && ((o + 1) % P) == 0;
    h->launches[K_SWEEPA]++;
    h->launches[K_SWEEPC]++;
    if (h->kind == KIND_CSR) { h->launches[K_SPMVB]++; h->launches[K_SPMVD]++; }
    if (rr) { h->launches[K_RR1]++; h->launches[K_RR2]++; }
    if (h->gap_on) h->launches[K_GAP]++;
  }
  return PBICG_OK;
}

void destroy_graphs(pbicg_ctx* h) {
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
}

pbicg_status ensure_hist(pbicg_ctx* h, int64_t need) {
  if (need <= h->hist_cap) return PBICG_OK;
  destroy_graphs(h);  // graphs captured the old pointers
  int64_t cap = need < 1024 ? 1024 : need;
  void *a = nullptr, *b = nullptr;
  pbicg_status st = dalloc(h, &a, (size_t)cap * sizeof(double));
  if (st) return st;
  st = dalloc(h, &b, (size_t)cap * sizeof(double));
  if (st) return st;
  h->hist.rnorm = (double*)a;
  h->hist.gap = (double*)b;
  h->hist_cap = cap;
  return PBICG_OK;
}

// Tile geometry of the TMA 2.5D sweeps (tile_sweeps.cuh): TY full x-lines per
// tile (3D) or one x-line (2D), a chunk of planes per work unit, units spread
// statically over one CTA per SM (deterministic accumulation order).
void setup_tile(pbicg_ctx* h) {
  const Geo& g = h->geo;
  TileGeo& t = h->tg;
  h->tile_ok = false;
  const int dim = h->dim;
  const int64_t tpmax = 2LL * TNT * TKMAX;
  if (g.nx > tpmax) return;
  const int64_t lines = dim == 3 ? g.ny : 1;
  int64_t TY = dim == 3 ? (1024 / g.nx) : 1;
  if (TY < 1) TY = 1;
  if (TY > lines) TY = lines;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
  const size_t reserve = 4096;  // static shared memory of the block reductions
  for (; TY >= 1; --TY) {
    t.nx = g.nx;
    t.ny = lines;
    t.nol = g.nol;
    t.o0 = g.o0;
    t.nog = g.nog;
    t.pxy = g.pxy;
    t.TY = (int32_t)TY;
    t.halo = (int32_t)(dim == 3 ? g.nx + 2 : 2);
    const int64_t TP = TY * g.nx;
    t.st_stride = (int32_t)((TP + 2 + 1) & ~1LL);
    t.sv_stride = (int32_t)((TP + 2 * t.halo + 2 + 1) & ~1LL);
    if (tile_smem_bytes(t, 1) + reserve <= (size_t)max_smem &&
        tile_smem_bytes(t, 0) + reserve <= (size_t)max_smem)
      break;
  }
  if (TY < 1) return;
  for (int i = 0; i < 7; ++i) t.c[i] = g.c[i];
  t.dinv = g.dinv;
  t.ncols = (int32_t)((lines + TY - 1) / TY);
  // chunk count: minimise the idle fraction of the last round of units
  const int grid = h->num_sm;
  int64_t best_n = 1;
  double best_w = 1e30;
  for (int64_t nch = 1; nch <= g.nol; ++nch) {
    const int64_t chunk = (g.nol + nch - 1) / nch;
    const int64_t nchk = (g.nol + chunk - 1) / chunk;
    const int64_t units = nchk * t.ncols;
    const int64_t rounds = (units + grid - 1) / grid;
    // work per CTA ~ rounds * (chunk + 2 prologue planes); ideal ~ units*chunk/grid
    const double w = (double)rounds * (double)(chunk + 2) * 1.0;
    if (w < best_w - 1e-9) {
      best_w = w;
      best_n = nch;
    }
    if (units > 64LL * grid) break;
  }
  t.chunk = (int32_t)((g.nol + best_n - 1) / best_n);
  t.nchunks = (int32_t)((g.nol + t.chunk - 1) / t.chunk);
  t.units = t.nchunks * t.ncols;
  h->tile_smem[0] = tile_smem_bytes(t, 0);
  h->tile_smem[1] = tile_smem_bytes(t, 1);
  cudaError_t e1, e2;
  if (dim == 3) {
    e1 = cudaFuncSetAttribute(t_sweep<3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)h->tile_smem[0]);
    e2 = cudaFuncSetAttribute(t_sweep<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)h->tile_smem[1]);
  } else {
    e1 = cudaFuncSetAttribute(t_sweep<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)h->tile_smem[0]);
    e2 = cudaFuncSetAttribute(t_sweep<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)h->tile_smem[1]);
  }
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  h->tile_ok = true;
}

pbicg_status common_setup(pbicg_ctx* h, void* cuda_stream) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(h, PBICG_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  CU(cudaGetDevice(&h->device));
  CU(cudaDeviceGetAttribute(&h->num_sm, cudaDevAttrMultiProcessorCount, h->device));
  if (cuda_stream) {
    h->stream = (cudaStream_t)cuda_stream;
  } else {
    CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  CU(cudaEventCreateWithFlags(&h->ev_entry, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_poll[0], cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_poll[1], cudaEventDisableTiming));
  void* p = nullptr;
  pbicg_status st = dalloc(h, &p, sizeof(Scal));
  if (st) return st;
  h->scal = (Scal*)p;
  CU(cudaMemsetAsync(h->scal, 0, sizeof(Scal), h->stream));
  CU(cudaMallocHost(&h->scal_host, 2 * sizeof(Scal)));
  return PBICG_OK;
}

// order the handle's stream after prior work on the legacy default stream
pbicg_status entry_sync(pbicg_ctx* h) {
  if (h->own_stream) {
    CU(cudaEventRecord(h->ev_entry, 0));
    CU(cudaStreamWaitEvent(h->stream, h->ev_entry, 0));
  }
  return PBICG_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

pbicg_status pbicgstab_create_stencil(const pbicg_stencil* op, pbicg_prec prec,
                                      const pbicg_dist* dist, void* cuda_stream,
                                      pbicg_handle* out) {
  pbicg_ctx* h = nullptr;
  if (!op || !out) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  *out = nullptr;
  if (prec != PBICG_PREC_JACOBI) return fail(nullptr, PBICG_EINVAL, "only Jacobi is supported");
  if (op->dim != 2 && op->dim != 3) return fail(nullptr, PBICG_EINVAL, "dim must be 2 or 3");
  int64_t nz = op->dim == 3 ? op->nz : 1;
  if (op->nx < 1 || op->ny < 1 || nz < 1) return fail(nullptr, PBICG_EINVAL, "grid sizes must be >= 1");
  if (op->coef[0] == 0.0 || !std::isfinite(op->coef[0]))
    return fail(nullptr, PBICG_EINVAL, "centre coefficient must be finite and nonzero (Jacobi)");
  for (int i = 0; i < 7; ++i)
    if (!std::isfinite(op->coef[i])) return fail(nullptr, PBICG_EINVAL, "non-finite coefficient");
  if (dist && dist->nranks > 1)
    return fail(nullptr, PBICG_ESTATE, "multi-GPU stencil path not available in this build");
  h = new pbicg_ctx();
  h->kind = KIND_STENCIL;
  h->dim = op->dim;
  pbicg_status st = common_setup(h, cuda_stream);
  if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  Geo& g = h->geo;
  g.nx = op->nx;
  g.ny = op->ny;
  if (op->dim == 3) {
    g.nog = nz;
    g.o0 = 0;
    g.nol = nz;
    g.pxy = op->nx * op->ny;
    g.nlines = op->ny * g.nol;
  } else {
    g.nog = op->ny;
    g.o0 = 0;
    g.nol = op->ny;
    g.pxy = op->nx;
    g.nlines = g.nol;
  }
  for (int i = 0; i < 7; ++i) g.c[i] = op->coef[i];
  if (op->dim == 2) { g.c[5] = 0.0; g.c[6] = 0.0; }
  g.dinv = 1.0 / op->coef[0];
  h->n_global = op->nx * op->ny * nz;
  h->n_local = g.nx * g.pxy / g.nx * g.nol;
  h->n_local = (op->dim == 3) ? g.pxy * g.nol : g.nx * g.nol;
  h->row_begin = g.o0 * g.pxy;
  h->H = g.pxy + g.nx + 4;  // ghost planes + staging slack of the tile kernels
  h->block = 256;
  if (g.nx < 256) h->block = (int)(((g.nx + 31) / 32) * 32);
  if (h->block < 64) h->block = 64;
  double** vs[] = {&h->V.x, &h->V.r, &h->V.rh, &h->V.k, &h->V.g, &h->V.s, &h->V.l, &h->V.b,
                   &h->V.w0, &h->V.w1, &h->V.z0, &h->V.z1, &h->V.zrr, &h->xtmp};
  for (double** v : vs) {
    st = gvec(h, v);
    if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  }
  int64_t L = g.nlines;
  if (op->dim == 3) {
    h->grid[K_INIT] = occ_grid(h, k_init1<3>, L);
    h->grid[K_SWEEPA] = occ_grid(h, k_sweepA<3>, L);
    h->grid[K_SWEEPC] = occ_grid(h, k_sweepC<3>, L);
    h->grid[K_RR1] = occ_grid(h, k_rr1<3>, L);
    h->grid[K_RR2] = occ_grid(h, k_rr2<3>, L);
    h->grid[K_GAP] = occ_grid(h, k_gap<3>, L);
    h->grid[K_APPLY] = occ_grid(h, k_apply<3>, L);
  } else {
    h->grid[K_INIT] = occ_grid(h, k_init1<2>, L);
    h->grid[K_SWEEPA] = occ_grid(h, k_sweepA<2>, L);
    h->grid[K_SWEEPC] = occ_grid(h, k_sweepC<2>, L);
    h->grid[K_RR1] = occ_grid(h, k_rr1<2>, L);
    h->grid[K_RR2] = occ_grid(h, k_rr2<2>, L);
    h->grid[K_GAP] = occ_grid(h, k_gap<2>, L);
    h->grid[K_APPLY] = occ_grid(h, k_apply<2>, L);
  }
  setup_tile(h);
  int gmax = h->num_sm;
  for (int k = 0; k < K_N; ++k) gmax = h->grid[k] > gmax ? h->grid[k] : gmax;
  void* p = nullptr;
  st = dalloc(h, &p, (size_t)gmax * 8 * sizeof(Dd));
  if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  h->part = (Dd*)p;
  st = ensure_hist(h, 1024);
  if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    g_create_err = cudaGetErrorString(e);
    pbicgstab_destroy(h);
    return PBICG_ECUDA;
  }
  *out = h;
  return PBICG_OK;
}

pbicg_status pbicgstab_create_csr(const pbicg_csr* op, pbicg_prec prec, const pbicg_dist* dist,
                                  void* cuda_stream, pbicg_handle* out) {
  pbicg_ctx* h = nullptr;
  if (!op || !out || !op->row_ptr || (!op->col && op->n_local > 0) || (!op->val && op->n_local > 0))
    return fail(nullptr, PBICG_EINVAL, "NULL argument");
  *out = nullptr;
  if (prec != PBICG_PREC_JACOBI) return fail(nullptr, PBICG_EINVAL, "only Jacobi is supported");
  const int64_t n = op->n_local;
  if (op->n_global < 1 || n < 1 || op->row_begin < 0 || op->row_begin + n > op->n_global)
    return fail(nullptr, PBICG_EINVAL, "bad row range");
  if (dist && dist->nranks > 1)
    return fail(nullptr, PBICG_ESTATE, "multi-GPU CSR path not available in this build");
  if (op->row_begin != 0 || n != op->n_global)
    return fail(nullptr, PBICG_EINVAL, "single GPU: the rank must own all rows");
  if (op->n_global > INT32_MAX) return fail(nullptr, PBICG_EINVAL, "n_global must fit int32");
  const int64_t* rp = op->row_ptr;
  int64_t width = 0;
  bool uniform = true;
  std::vector<double> dinv(n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t len = rp[i + 1] - rp[i];
    if (len < 1) return fail(nullptr, PBICG_EINVAL, "row without entries (needs a diagonal)");
    if (i > 0 && len != width) uniform = false;
    if (len > width) width = len;
    bool diag = false;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t c = op->col[p];
      if (c < 0 || c >= op->n_global) return fail(nullptr, PBICG_EINVAL, "column out of range");
      if (p > rp[i] && c <= op->col[p - 1])
        return fail(nullptr, PBICG_EINVAL, "columns must be strictly ascending within a row");
      if (!std::isfinite(op->val[p])) return fail(nullptr, PBICG_EINVAL, "non-finite value");
      if (c == op->row_begin + i) {
        if (op->val[p] == 0.0) return fail(nullptr, PBICG_EINVAL, "zero diagonal (Jacobi undefined)");
        dinv[i] = 1.0 / op->val[p];  // A3
        diag = true;
      }
    }
    if (!diag) return fail(nullptr, PBICG_EINVAL, "missing diagonal entry");
  }
  if (width > 4096) return fail(nullptr, PBICG_EINVAL, "row too long for the ELL path (> 4096)");
  h = new pbicg_ctx();
  h->kind = KIND_CSR;
  pbicg_status st = common_setup(h, cuda_stream);
  if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  h->n_global = op->n_global;
  h->n_local = n;
  h->row_begin = op->row_begin;
  h->H = 0;
  h->block = 256;
  // column-major ELL in stored row order; padding slots are never read (len[])
  std::vector<int32_t> ecol((size_t)width * n);
  std::vector<double> eval((size_t)width * n, 0.0);
  std::vector<int32_t> elen(uniform ? 0 : n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t len = rp[i + 1] - rp[i];
    if (!uniform) elen[i] = (int32_t)len;
    for (int64_t q = 0; q < width; ++q) {
      bool real = q < len;
      ecol[(size_t)q * n + i] = real ? (int32_t)(op->col[rp[i] + q] - op->row_begin) : (int32_t)i;
      eval[(size_t)q * n + i] = real ? op->val[rp[i] + q] : 0.0;
    }
  }
  void *pc = nullptr, *pv = nullptr, *pl = nullptr, *pd = nullptr;
  if ((st = dalloc(h, &pc, ecol.size() * sizeof(int32_t))) ||
      (st = dalloc(h, &pv, eval.size() * sizeof(double))) ||
      (st = dalloc(h, &pd, (size_t)n * sizeof(double)))) {
    g_create_err = h->err; pbicgstab_destroy(h); return st;
  }
  if (!uniform && (st = dalloc(h, &pl, (size_t)n * sizeof(int32_t)))) {
    g_create_err = h->err; pbicgstab_destroy(h); return st;
  }
  cudaError_t e = cudaMemcpy(pc, ecol.data(), ecol.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(pv, eval.data(), eval.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(pd, dinv.data(), (size_t)n * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !uniform)
    e = cudaMemcpy(pl, elen.data(), (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    g_create_err = cudaGetErrorString(e);
    pbicgstab_destroy(h);
    return PBICG_ECUDA;
  }
  h->csr.n = n;
  h->csr.width = (int32_t)width;
  h->csr.col = (const int32_t*)pc;
  h->csr.val = (const double*)pv;
  h->csr.len = uniform ? nullptr : (const int32_t*)pl;
  h->csr.dinv = (const double*)pd;
  double** vs[] = {&h->V.x, &h->V.r, &h->V.rh, &h->V.k, &h->V.g, &h->V.s, &h->V.l, &h->V.b,
                   &h->V.w0, &h->V.w1, &h->V.z0, &h->V.z1, &h->V.zrr, &h->xtmp};
  for (double** v : vs) {
    st = gvec(h, v);
    if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  }
  const int64_t blocks = (n + h->block - 1) / h->block;
  h->grid[K_INIT] = occ_grid(h, c_init1, blocks);
  h->grid[K_SWEEPA] = occ_grid(h, c_sweepA, blocks);
  h->grid[K_SWEEPC] = occ_grid(h, c_sweepC, blocks);
  h->grid[K_SPMVB] = occ_grid(h, c_spmvB, blocks);
  h->grid[K_SPMVD] = occ_grid(h, c_spmvD, blocks);
  h->grid[K_RR1] = occ_grid(h, c_rr1, blocks);
  h->grid[K_RR2] = occ_grid(h, c_rr2, blocks);
  h->grid[K_GAP] = occ_grid(h, c_gap, blocks);
  h->grid[K_APPLY] = occ_grid(h, c_apply, blocks);
  int gmax = 0;
  for (int k = 0; k < K_N; ++k) gmax = h->grid[k] > gmax ? h->grid[k] : gmax;
  void* p = nullptr;
  st = dalloc(h, &p, (size_t)gmax * 8 * sizeof(Dd));
  if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  h->part = (Dd*)p;
  st = ensure_hist(h, 1024);
  if (st) { g_create_err = h->err; pbicgstab_destroy(h); return st; }
  e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    g_create_err = cudaGetErrorString(e);
    pbicgstab_destroy(h);
    return PBICG_ECUDA;
  }
  *out = h;
  return PBICG_OK;
}

pbicg_status pbicgstab_local_rows(pbicg_handle h, int64_t* row_begin, int64_t* n_local) {
  if (!h) return fail(nullptr, PBICG_EINVAL, "NULL handle");
  if (row_begin) *row_begin = h->row_begin;
  if (n_local) *n_local = h->n_local;
  return PBICG_OK;
}

pbicg_status pbicgstab_set_option(pbicg_handle h, const char* key, int64_t value) {
  if (!h || !key) return fail(h, PBICG_EINVAL, "NULL argument");
  std::string k(key);
  if (k == "bench") h->bench = value != 0;
  else if (k == "graphs") h->use_graphs = value != 0;
  else if (k == "timing") h->timing = value != 0;
  else if (k == "overlap") h->overlap = value != 0;
  else if (k == "tile") {
    h->tile_on = value != 0;
    destroy_graphs(h);
  }
  else if (k == "schedule") {
    if (value < 0 || value > 2) return fail(h, PBICG_EINVAL, "schedule must be 0, 1 or 2");
    if (value == 1 && h->kind == KIND_CSR) return fail(h, PBICG_EINVAL, "fused schedule is stencil-only");
    h->schedule = (int)value;
  } else return fail(h, PBICG_EINVAL, "unknown option '" + k + "'");
  return PBICG_OK;
}

pbicg_status pbicgstab_apply(pbicg_handle h, const double* x_dev, double* y_dev) {
  if (!h || !x_dev || !y_dev) return fail(h, PBICG_EINVAL, "NULL argument");
  pbicg_status st = entry_sync(h);
  if (st) return st;
  CU(cudaMemcpyAsync(h->xtmp, x_dev, (size_t)h->n_local * sizeof(double),
                     cudaMemcpyDeviceToDevice, h->stream));
  {
    LaunchScope ls(h, K_APPLY);
    if (h->kind == KIND_CSR)
      c_apply<<<h->grid[K_APPLY], h->block, 0, h->stream>>>(h->csr, h->xtmp, y_dev);
    else if (h->dim == 3)
      k_apply<3><<<h->grid[K_APPLY], h->block, 0, h->stream>>>(h->geo, h->xtmp, y_dev);
    else
      k_apply<2><<<h->grid[K_APPLY], h->block, 0, h->stream>>>(h->geo, h->xtmp, y_dev);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->stream));
  if (h->timing) collect_timing(h);
  return PBICG_OK;
}

pbicg_status pbicgstab_solve(pbicg_handle h, const double* b_dev, const double* x0_dev,
                             double tol, int32_t maxit, int32_t rr_period, double* x_dev_out,
                             double* rnorm_hist, double* gap_hist, int32_t* iters_out,
                             int32_t* outcome_out) {
  if (!h) return fail(nullptr, PBICG_EINVAL, "NULL handle");
  if (h->failed) return fail(h, PBICG_ESTATE, "handle is in a failed state");
  if (!b_dev || !x0_dev || !x_dev_out || !rnorm_hist || !iters_out || !outcome_out)
    return fail(h, PBICG_EINVAL, "NULL argument");
  if (maxit < 0 || rr_period < 0 || !(tol >= 0.0))
    return fail(h, PBICG_EINVAL, "maxit, rr_period and tol must be >= 0");
  pbicg_status st = ensure_hist(h, (int64_t)maxit + 1);
  if (st) return st;
  st = entry_sync(h);
  if (st) return st;
  h->gap_on = gap_hist != nullptr;
  const size_t nb = (size_t)h->n_local * sizeof(double);
  CU(cudaMemcpyAsync(h->V.b, b_dev, nb, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaMemcpyAsync(h->V.x, x0_dev, nb, cudaMemcpyDeviceToDevice, h->stream));
  // A1: g, s, l, z_{-1} (and the spare buffers) start at zero
  double* zs[] = {h->V.g, h->V.s, h->V.l, h->V.z0, h->V.z1, h->V.zrr};
  for (double* v : zs) CU(cudaMemsetAsync(v - h->H, 0, nb + 2 * h->H * sizeof(double), h->stream));
  Scal s0;
  memset(&s0, 0, sizeof(s0));
  s0.tol = tol;
  s0.sqrt_eps = std::sqrt(std::ldexp(1.0, -53));
  s0.outcome = OUT_MAXIT;
  s0.gap_iter = -1;
  s0.bench = h->bench;
  s0.rr_period = rr_period;
  *h->scal_host = s0;
  CU(cudaMemcpyAsync(h->scal, h->scal_host, sizeof(Scal), cudaMemcpyHostToDevice, h->stream));
  enq_init(h);
  CU(cudaGetLastError());
  // chunk length: a multiple of the replacement period so every chunk has the
  // same replacement pattern (A11)
  int P = rr_period;
  int L = 32;
  if (P > 0) L = P >= 32 ? P : P * ((32 + P - 1) / P);
  int64_t done_its = 0;
  int slot = 0;
  bool have_prev = false;
  bool stop = false;
  while (done_its < maxit && !stop) {
    int n = (int)((maxit - done_its) < L ? (maxit - done_its) : L);
    st = run_chunk(h, n, P);
    if (st) { h->failed = true; return st; }
    done_its += n;
    // async poll: copy the state, check the previous chunk's copy
    CU(cudaMemcpyAsync(h->scal_host + slot, h->scal, sizeof(Scal), cudaMemcpyDeviceToHost,
                       h->stream));
    CU(cudaEventRecord(h->ev_poll[slot], h->stream));
    if (have_prev) {
      CU(cudaEventSynchronize(h->ev_poll[slot ^ 1]));
      if (h->scal_host[slot ^ 1].done) stop = true;
    }
    have_prev = true;
    slot ^= 1;
  }
  CU(cudaStreamSynchronize(h->stream));
  CU(cudaMemcpy(h->scal_host, h->scal, sizeof(Scal), cudaMemcpyDeviceToHost));
  const Scal& S = *h->scal_host;
  int32_t iters = S.done ? S.iters : S.iter;
  if (S.done && S.outcome == OUT_BREAKDOWN) iters = S.iters;
  if (iters > maxit) iters = maxit;
  CU(cudaMemcpy(rnorm_hist, h->hist.rnorm, (size_t)(iters + 1) * sizeof(double),
                cudaMemcpyDeviceToHost));
  if (gap_hist)
    CU(cudaMemcpy(gap_hist, h->hist.gap, (size_t)(iters + 1) * sizeof(double),
                  cudaMemcpyDeviceToHost));
  CU(cudaMemcpyAsync(x_dev_out, h->V.x, nb, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (h->timing) collect_timing(h);
  *iters_out = iters;
  *outcome_out = S.done ? S.outcome : OUT_MAXIT;
  return PBICG_OK;
}

pbicg_status pbicgstab_solve_host(pbicg_handle h, const double* b_host, const double* x0_host,
                                  double tol, int32_t maxit, int32_t rr_period,
                                  double* x_host_out, double* rnorm_hist, double* gap_hist,
                                  int32_t* iters_out, int32_t* outcome_out) {
  if (!h) return fail(nullptr, PBICG_EINVAL, "NULL handle");
  if (!b_host || !x0_host || !x_host_out) return fail(h, PBICG_EINVAL, "NULL argument");
  const size_t nb = (size_t)h->n_local * sizeof(double);
  pbicg_status st = entry_sync(h);
  if (st) return st;
  // stage through the handle's own buffers: b -> V.b, x0 -> xtmp
  CU(cudaMemcpyAsync(h->xtmp, x0_host, nb, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(h->V.rh, b_host, nb, cudaMemcpyHostToDevice, h->stream));
  st = pbicgstab_solve(h, h->V.rh, h->xtmp, tol, maxit, rr_period, h->xtmp, rnorm_hist,
                       gap_hist, iters_out, outcome_out);
  if (st) return st;
  CU(cudaMemcpy(x_host_out, h->xtmp, nb, cudaMemcpyDeviceToHost));
  return PBICG_OK;
}

pbicg_status pbicgstab_kernel_time(pbicg_handle h, const char* name, int64_t* launches, double* ms,
                                   int32_t reset) {
  if (!h || !name) return fail(h, PBICG_EINVAL, "NULL argument");
  std::string n(name);
  int64_t L = 0;
  double t = 0;
  bool found = false;
  for (int k = 0; k < K_N; ++k) {
    if (n == "all" || n == kname_str[k]) {
      L += h->launches[k];
      t += h->ms[k];
      found = true;
    }
  }
  if (!found) return fail(h, PBICG_EINVAL, "unknown kernel name '" + n + "'");
  if (launches) *launches = L;
  if (ms) *ms = h->timing ? t : NAN;
  if (reset) {
    for (int k = 0; k < K_N; ++k) { h->launches[k] = 0; h->ms[k] = 0; }
  }
  return PBICG_OK;
}

pbicg_status pbicgstab_kernel_bytes(pbicg_handle h, const char* name, double* bytes) {
  if (!h || !name || !bytes) return fail(h, PBICG_EINVAL, "NULL argument");
  std::string n(name);
  const double N = (double)h->n_local;
  double b = 0;
  if (h->kind == KIND_STENCIL) {
    // fused schedule: streams read + written once per launch (DESIGN.md Roofline)
    if (n == "sweepA") b = 11 * 8 * N;       // read k,g,l,w,s,z,r; write g,s,l,z
    else if (n == "sweepC") b = 13 * 8 * N;  // read x,g,k,l,r,s,w,z,r^; write x,r,k,w
    else if (n == "rr1") b = 7 * 8 * N;      // read x,b,g; write r,k,s,l
    else if (n == "rr2") b = 5 * 8 * N;      // read r,s,r^; write w,z
    else if (n == "gap") b = 3 * 8 * N;
    else if (n == "apply") b = 2 * 8 * N;
    else if (n == "iteration") b = 24 * 8 * N;
  } else {
    const double nnz = (double)h->csr.width;  // ELL width
    const double mat = 12.0 * nnz * N;        // val (8) + col (4) per slot
    if (n == "sweepA") b = 14 * 8 * N;        // read k,g,l,w,s,z,t,v,r,dinv; write g,s,l,z
    else if (n == "spmvB" || n == "spmvD" || n == "apply") b = mat + 3 * 8 * N;  // in, dinv, out
    else if (n == "sweepC") b = 16 * 8 * N;   // read x,g,k,l,r,s,w,z,t,v,r^,dinv; write x,r,k,w
    else if (n == "rr1") b = 2 * mat + 8 * 8 * N;
    else if (n == "rr2") b = 2 * mat + 7 * 8 * N;
    else if (n == "gap") b = mat + 3 * 8 * N;
    else if (n == "iteration") b = 2 * mat + 36 * 8 * N;
  }
  *bytes = b;
  return PBICG_OK;
}

pbicg_status pbicgstab_get_unique_id(void* out128) {
  (void)out128;
  return fail(nullptr, PBICG_ESTATE, "NCCL support not built");
}

const char* pbicgstab_last_error(pbicg_handle h) {
  return h ? h->err.c_str() : g_create_err.c_str();
}

void pbicgstab_destroy(pbicg_handle h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  collect_timing(h);
  destroy_graphs(h);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  for (void* p : h->allocs) cudaFree(p);
  if (h->scal_host) cudaFreeHost(h->scal_host);
  if (h->ev_entry) cudaEventDestroy(h->ev_entry);
  if (h->ev_poll[0]) cudaEventDestroy(h->ev_poll[0]);
  if (h->ev_poll[1]) cudaEventDestroy(h->ev_poll[1]);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  cudaGetLastError();
  delete h;
}

}  // extern "C"
