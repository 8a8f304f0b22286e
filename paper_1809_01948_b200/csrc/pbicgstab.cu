// pbicgstab.cu -- host driver and C ABI (include/pbicgstab.h) of the B200
// p-BiCGStab library.  One translation unit, compiled with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
// (no FMA contraction anywhere: reading A4).
//
// Host responsibilities only: validation, partitioning, workspace allocation,
// launch order, the rank exchange (NCCL across processes, or the loopback
// transport that emulates P ranks inside one process), CUDA-graph capture/replay
// of chunks of iterations, asynchronous polling of the device `done` flag,
// history download.  Every arithmetic step of Alg. 2 runs in the kernels of
// stencil_kernels.cuh / tile_sweeps.cuh / csr_kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/pbicgstab.h"
#include "csr_kernels.cuh"
#include "ilu_kernels.cuh"
#include "nccl_dyn.h"
#include "stencil_kernels.cuh"
#include "tile_bj.h"
#include "tile_jac.h"
#include "tile_seg.h"
#include "tile_sweeps.cuh"
#include "spmv_tile.cuh"

namespace {

thread_local std::string g_create_err;
constexpr int WIN_SMEM = 64 + WRS * (int)sizeof(double);

enum Kname { K_INIT = 0, K_SWEEPA, K_SWEEPC, K_SPMVB, K_SPMVD, K_RR1, K_RR2, K_GAP, K_APPLY, K_FIN,
             K_CL1, K_CL2, K_CL3, K_PC, K_PREC, K_N };
const char* kname_str[K_N] = {"init", "sweepA", "sweepC", "spmvB", "spmvD", "rr1", "rr2", "gap",
                              "apply", "fin", "cl1", "cl2", "cl3", "pcg", "prec"};

// solver selected with option "method"
enum Method { M_PBICGSTAB = 0, M_BICGSTAB = 1, M_PIPECG = 2 };

// tile modes that have a block-Jacobi instance (p-BiCGStab + automated replacement;
// the raw-stencil gap kernel needs none; the comparison solvers use Jacobi only)
constexpr bool bj_mode(int m) {
  return m == TM_A || m == TM_C || m == TM_RR1 || m == TM_RR2 || m == TM_INIT1 ||
         m == TM_INIT2 || m == TM_AN || m == TM_CN || m == TM_RR1N || m == TM_RR2N ||
         m == TM_INIT1N || m == TM_CL1 || m == TM_CL2 || m == TM_CL3 || m == TM_PC ||
         m == TM_PCI1 || m == TM_PCI2;
}

struct TimedLaunch {
  int k;
  cudaEvent_t e0, e1;
};

enum Kind { KIND_STENCIL = 0, KIND_CSR = 1 };
enum Comm { COMM_NONE = 0, COMM_NCCL = 1, COMM_LOOP = 2 };

}  // namespace

struct pbicg_group;

struct pbicg_ctx {
  int kind = KIND_STENCIL;
  int dim = 3;
  int device = 0, num_sm = 0;
  cudaStream_t stream = nullptr, side = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_entry = nullptr, ev_poll[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t n_local = 0, row_begin = 0, n_global = 0, H = 0;
  int64_t halo_n = 0;  // rows exchanged per side with each neighbour
  Geo geo{};
  TileGeo tg{};
  bool tile_ok = false;  // TMA 2.5D sweeps eligible for this operator
  bool tile_vec = false; // ... with 16-byte aligned pairs (nx even)
  // split schedule's stand-alone SpMVs on tall tiles (spmv_tile.cuh; 3D Jacobi, nx even)
  // light steps on tall tiles (spmv_tile.cuh; 3D Jacobi, nx even): the split
  // schedule's stand-alone SpMVs (4 row pairs per thread) and the replacement step (2)
  bool spt_ok = false, lrr_ok = false;
  size_t spt_smem = 0, lrr_smem = 0;
  SpmvGeo sq{}, sq_rr{};
  bool tile_seg = false; // ... as x-segmented tiles (nx > 1024, or 3D planes too wide for
                         // full-line tiles; instances in tile_seg.cu)
  int tile_on = 1;       // option "tile"
  size_t tile_smem[TM_N] = {0};
  int tile_occ[TM_N] = {0};  // resident CTAs per SM of each tile kernel
  CsrOp csr{};
  WinGeo wg{};
  bool win_ok = false;  // banded CSR: window SpMV (c_spmv_win) eligible
  int win_grid = 0;
  bool cst_ok = false;  // CSR: TMA-staged sweeps (c_sweep_tma) eligible (Jacobi)
  bool cst_on = true;   // option "csr_tma"
  // ILU(0) / ICC(0) preconditioner (reading A34): factors of this rank's diagonal block
  int ilu = 0;          // 1 ILU(0), 2 ICC(0) (symmetric A)
  bool ilu_st = false;  // stencil wavefront kernels (else the general CSR level-order kernel)
  IluOp ilu_op{};
  int ilu_grid = 0;
  int cst_grid = 0;
  std::vector<void*> allocs;
  Vecs V{};
  double* xtmp = nullptr;    // ghosted scratch (apply input, host-solve staging)
  double* dinv_g = nullptr;  // CSR: ghosted dinv
  Scal* scal = nullptr;
  Scal* scal_host = nullptr;  // pinned [2] (poll double buffer)
  Dd* part = nullptr;
  Dd *red_send = nullptr, *red_recv = nullptr;
  Hist hist{nullptr, nullptr};
  int64_t hist_cap = 0;
  int block = 256;
  int grid[16] = {0};
  // distribution
  int nranks = 1, rank = 0;
  bool dist = false;  // rank-row exchange path: nranks > 1, or an NCCL communicator of 1 rank
  int comm = COMM_NONE;
  ncclComm_t nccl_halo = nullptr, nccl_red = nullptr;
  pbicg_group* group = nullptr;
  // options
  int bench = 0, use_graphs = 1, timing = 0, overlap = 1, schedule = 0, gap_on = 0;
  bool auto_split = false;  // schedule 0 picks the split schedule (NCCL ranks, small slabs)
  int method = M_PBICGSTAB;
  int auto_rr = 0;                           // option rr_auto
  double ar_nA = 0, ar_muN = 0, ar_mutN = 0;  // bound constants (reading A29)
  bool ar_ok = false;                        // constants known for this operator
  int32_t last_iters = -1;                   // iterations of the last solve
  int grid_a2 = 0, grid_c2 = 0;              // split stencil schedule sweeps (occupancy grids)
  // peer-memory reduction transport (option "transport" 1; state.cuh publish/k_fin)
  int p2p = 0;
  Dd* p2p_buf = nullptr;                     // own receive buffer [2][nranks][RED_K]
  unsigned long long* p2p_flags = nullptr;   // own flags [nranks]
  unsigned long long* p2p_ep = nullptr;      // own epoch counter
  std::vector<Dd*> p2p_recv_tab;             // every rank's buffer, in this address space
  std::vector<unsigned long long*> p2p_flag_tab;
  std::vector<void*> ipc_opened;             // peer mappings to close
  // transport 1, fused schedule: neighbours' ghost planes of w0, w1, z0, z1 ([q][0]:
  // the lower neighbour's upper ghost, [q][1]: the upper neighbour's lower ghost)
  double* peer_ghost[4][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr},
                              {nullptr, nullptr}};
  int64_t halo_ops = 0;  // halo exchanges enqueued (copies / NCCL groups), for tests
  int32_t last_nrr = 0;                      // replacements of the last solve
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs;
  std::vector<TimedLaunch> pending;
  std::vector<cudaEvent_t> ev_pool;
  int64_t launches[16] = {0};
  double ms[16] = {0};
  bool failed = false;
  std::string err;
};

// P handles emulating P ranks in one process on one device (loopback transport).
struct pbicg_group {
  std::vector<pbicg_ctx*> m;
  int alive = 0;
};

using Members = std::vector<pbicg_ctx*>;

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

#define NC(call)                                                      \
  do {                                                                \
    ncclResult_t r_ = (call);                                         \
    if (r_ != ncclSuccess) {                                          \
      return fail(h, PBICG_ENCCL,                                     \
                  std::string(#call) + ": " + nccl_api().GetErrorString(r_)); \
    }                                                                 \
  } while (0)

#define ST(call)                   \
  do {                             \
    pbicg_status s_ = (call);      \
    if (s_ != PBICG_OK) return s_; \
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
  size_t n = (size_t)(h->n_local + 2 * h->H) + 2;  // +2: 16-byte rounding of bulk copies
  ST(dalloc(h, &p, n * sizeof(double)));
  CU(cudaMemsetAsync(p, 0, n * sizeof(double), h->stream));
  *out = (double*)p + h->H;
  return PBICG_OK;
}

// Create-time host->device upload.  Every create-time write goes through the
// handle's stream (a cudaStreamNonBlocking stream when the caller passes NULL),
// and the stream is drained before the call returns: a plain cudaMemcpy runs on
// the legacy default stream, which is NOT ordered against that stream, so it
// could land before gvec()'s zero-fill of the same buffer (dinv_g).
pbicg_status upload(pbicg_ctx* h, void* dst, const void* src, size_t bytes) {
  CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
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

Members members(pbicg_ctx* h) {
  if (h->comm == COMM_LOOP && h->group) return h->group->m;
  return Members{h};
}

// ---------------------------------------------------------------------------
// Kernel launches (one rank)
enum Phase { PH_INIT1, PH_INIT2, PH_SWEEPA, PH_SPMVB, PH_SWEEPC, PH_RR1, PH_RR2, PH_SPMVD, PH_GAP,
             PH_CL1, PH_CL2, PH_CL3, PH_PC, PH_PCI1, PH_PCI2,
             // CSR comparison solvers: element-wise steps and SpMVs with epilogues
             PH_CCP, PH_SP_CLS, PH_CCU, PH_SP_CLY, PH_CCX, PH_SP_PCW0, PH_SP_PCN, PH_CPC,
             PH_PRECMV,
             // stencil split schedule (option schedule 2)
             PH_SWEEPA2, PH_SWEEPC2, PH_SPB, PH_SPD };

template <int DIM, int MODE>
void launch_tile(pbicg_ctx* h) {
  int per_sm = h->tile_occ[MODE] > 0 ? h->tile_occ[MODE] : 1;
  if (Stash<MODE>::w || Stash<MODE>::r) {  // RR1 and RR2 on the same grid (the stash)
    const int a = h->tile_occ[BaseOf<MODE>::v != MODE ? TM_RR1N : TM_RR1];
    const int b = h->tile_occ[BaseOf<MODE>::v != MODE ? TM_RR2N : TM_RR2];
    per_sm = a < b ? a : b;
    if (per_sm < 1) per_sm = 1;
  }
  const int cap = h->num_sm * per_sm;
  const int grid = h->tg.units < cap ? h->tg.units : cap;
  if (h->tile_seg) {  // x-segmented instances live in tile_seg.cu
    tile_seg_launch(DIM, MODE, grid, h->tile_smem[MODE], h->stream, h->tg, h->V, h->scal,
                    h->part, h->hist);
    return;
  }
  if constexpr (bj_mode(MODE)) {  // block Jacobi instances live in tile_bj.cu
    const size_t sm = h->tile_smem[MODE];
    switch (h->tg.bj) {
      case 2: tile_bj_launch_2(DIM, MODE, grid, sm, h->stream, h->tg, h->V, h->scal, h->part, h->hist); return;
      case 4: tile_bj_launch_4(DIM, MODE, grid, sm, h->stream, h->tg, h->V, h->scal, h->part, h->hist); return;
      case 8: tile_bj_launch_8(DIM, MODE, grid, sm, h->stream, h->tg, h->V, h->scal, h->part, h->hist); return;
      default: break;
    }
  }
  // Jacobi instances live in tile_jac.cu (one object per pairing mode)
  if (h->tile_vec)
    tile_jac_launch_1(DIM, MODE, grid, h->tile_smem[MODE], h->stream, h->tg, h->V, h->scal,
                      h->part, h->hist);
  else
    tile_jac_launch_0(DIM, MODE, grid, h->tile_smem[MODE], h->stream, h->tg, h->V, h->scal,
                      h->part, h->hist);
}

template <int MODE>
void launch_light(pbicg_ctx* h);  // spmv_tile.cuh instances (below, with setup_light_tiles)

template <int DIM>
void launch_stencil(pbicg_ctx* h, Phase p) {
  const Geo& g = h->geo;
  const bool tile = h->tile_ok && h->tile_on;
  switch (p) {
    case PH_INIT1: {
      LaunchScope ls(h, K_INIT);
      if (h->auto_rr) launch_tile<DIM, TM_INIT1N>(h);
      else if (tile) launch_tile<DIM, TM_INIT1>(h);
      else k_init1<DIM><<<h->grid[K_INIT], h->block, 0, h->stream>>>(g, h->V, h->scal, h->part, h->hist);
    } break;
    case PH_INIT2: {
      LaunchScope ls(h, K_INIT);
      if (tile) launch_tile<DIM, TM_INIT2>(h);
      else k_init2<DIM><<<h->grid[K_INIT], h->block, 0, h->stream>>>(g, h->V, h->scal, h->part, h->hist);
    } break;
    case PH_SWEEPA: {
      LaunchScope ls(h, K_SWEEPA);
      if (h->auto_rr) launch_tile<DIM, TM_AN>(h);
      else if (tile) launch_tile<DIM, TM_A>(h);
      else k_sweepA<DIM><<<h->grid[K_SWEEPA], h->block, 0, h->stream>>>(g, h->V, h->scal, h->part,
                                                                          h->hist);
    } break;
    case PH_SWEEPC: {
      LaunchScope ls(h, K_SWEEPC);
      if (h->auto_rr) launch_tile<DIM, TM_CN>(h);
      else if (tile) launch_tile<DIM, TM_C>(h);
      else k_sweepC<DIM><<<h->grid[K_SWEEPC], h->block, 0, h->stream>>>(g, h->V, h->scal, h->part,
                                                                          h->hist);
    } break;
    case PH_RR1: {
      LaunchScope ls(h, K_RR1);
      if (h->auto_rr) launch_tile<DIM, TM_RR1N>(h);
      else if (DIM == 3 && tile && h->lrr_ok) launch_light<TM_RR1>(h);
      else if (tile) launch_tile<DIM, TM_RR1>(h);
      else k_rr1<DIM><<<h->grid[K_RR1], h->block, 0, h->stream>>>(g, h->V, h->scal);
    } break;
    case PH_RR2: {
      LaunchScope ls(h, K_RR2);
      if (h->auto_rr) launch_tile<DIM, TM_RR2N>(h);
      else if (DIM == 3 && tile && h->lrr_ok) launch_light<TM_RR2>(h);
      else if (tile) launch_tile<DIM, TM_RR2>(h);
      else k_rr2<DIM><<<h->grid[K_RR2], h->block, 0, h->stream>>>(g, h->V, h->scal, h->part, h->hist);
    } break;
    case PH_GAP: {
      LaunchScope ls(h, K_GAP);
      if (tile) launch_tile<DIM, TM_GAP>(h);
      else k_gap<DIM><<<h->grid[K_GAP], h->block, 0, h->stream>>>(g, h->V, h->scal, h->part, h->hist);
    } break;
    // comparison solvers: TMA tile kernels only (set_option("method") checks tile_ok)
    case PH_CL1: { LaunchScope ls(h, K_CL1); launch_tile<DIM, TM_CL1>(h); } break;
    case PH_CL2: { LaunchScope ls(h, K_CL2); launch_tile<DIM, TM_CL2>(h); } break;
    case PH_CL3: { LaunchScope ls(h, K_CL3); launch_tile<DIM, TM_CL3>(h); } break;
    case PH_PC: { LaunchScope ls(h, K_PC); launch_tile<DIM, TM_PC>(h); } break;
    case PH_PCI1: { LaunchScope ls(h, K_INIT); launch_tile<DIM, TM_PCI1>(h); } break;
    case PH_PCI2: { LaunchScope ls(h, K_INIT); launch_tile<DIM, TM_PCI2>(h); } break;
    case PH_SWEEPA2: {
      LaunchScope ls(h, K_SWEEPA);
      if (h->cst_ok && h->cst_on)  // TMA chunk ring (option csr_tma covers it too)
        c_sweep_tma<0, false, false, true><<<h->cst_grid, CST_T, kCstSmem, h->stream>>>(
            h->csr, h->V, h->scal, h->part, h->hist, g.dinv);
      else
        k_sweepA2<DIM><<<h->grid_a2, 256, 0, h->stream>>>(g, h->V, h->scal, h->part, h->hist);
    } break;
    case PH_SWEEPC2: {
      LaunchScope ls(h, K_SWEEPC);
      if (h->cst_ok && h->cst_on)
        c_sweep_tma<1, false, false, true><<<h->cst_grid, CST_T, kCstSmem, h->stream>>>(
            h->csr, h->V, h->scal, h->part, h->hist, g.dinv);
      else
        k_sweepC2<DIM><<<h->grid_c2, 256, 0, h->stream>>>(g, h->V, h->scal, h->part, h->hist);
    } break;
    case PH_SPB: {
      LaunchScope ls(h, K_SPMVB);
      if (DIM == 3 && h->spt_ok) launch_light<TM_SPB>(h);
      else launch_tile<DIM, TM_SPB>(h);
    } break;
    case PH_SPD: {
      LaunchScope ls(h, K_SPMVD);
      if (DIM == 3 && h->spt_ok) launch_light<TM_SPD>(h);
      else launch_tile<DIM, TM_SPD>(h);
    } break;
    default:
      break;
  }
}

template <int M>
void launch_spmv(pbicg_ctx* h) {
  if (h->win_ok)
    c_spmv_win<M><<<h->win_grid, WNT, WIN_SMEM, h->stream>>>(h->csr, h->V, h->scal, h->wg, h->part,
                                                             h->hist);
  else
    c_spmv_g<M><<<h->grid[K_SPMVB], h->block, 0, h->stream>>>(h->csr, h->V, h->scal, h->part,
                                                              h->hist);
}

// preconditioner kind of the per-row CSR kernels (csr_kernels.cuh PK_*)
int pk_of(const pbicg_ctx* h) { return h->ilu ? PK_ILU : (h->csr.bj > 1 ? PK_BJ : PK_JAC); }

// the per-row kernels, one instance per preconditioner kind (NRM: automated replacement,
// never with ILU(0))
template <int PK>
void launch_csr_rows(pbicg_ctx* h, Phase p) {
  const CsrOp& A = h->csr;
  const bool nrm = PK != PK_ILU && h->auto_rr;
  cudaStream_t st = h->stream;
  switch (p) {
    case PH_CCP: c_cl_p<PK><<<h->grid[K_SWEEPA], h->block, 0, st>>>(A, h->V, h->scal); break;
    case PH_CCU: c_cl_u<PK><<<h->grid[K_SWEEPA], h->block, 0, st>>>(A, h->V, h->scal); break;
    case PH_PRECMV: c_prec_mv<PK><<<h->grid[K_SWEEPA], h->block, 0, st>>>(A, h->V); break;
    case PH_CPC: c_pc<PK><<<h->grid[K_SWEEPC], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist); break;
    case PH_INIT1:
      if (nrm) c_init1<true, PK><<<h->grid[K_INIT], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      else c_init1<false, PK><<<h->grid[K_INIT], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      break;
    case PH_INIT2: c_init2<PK><<<h->grid[K_INIT], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist); break;
    case PH_SWEEPA:
      if (nrm) c_sweepA<true, PK><<<h->grid[K_SWEEPA], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      else c_sweepA<false, PK><<<h->grid[K_SWEEPA], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      break;
    case PH_SWEEPC:
      if (nrm) c_sweepC<true, PK><<<h->grid[K_SWEEPC], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      else c_sweepC<false, PK><<<h->grid[K_SWEEPC], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      break;
    case PH_RR1:
      if (nrm) c_rr1<true, PK><<<h->grid[K_RR1], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      else c_rr1<false, PK><<<h->grid[K_RR1], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      break;
    case PH_RR2:
      if (nrm) c_rr2<true, PK><<<h->grid[K_RR2], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      else c_rr2<false, PK><<<h->grid[K_RR2], h->block, 0, st>>>(A, h->V, h->scal, h->part, h->hist);
      break;
    default:
      break;
  }
}

void launch_rows(pbicg_ctx* h, Phase p) {
  switch (pk_of(h)) {
    case PK_ILU: launch_csr_rows<PK_ILU>(h, p); break;
    case PK_BJ: launch_csr_rows<PK_BJ>(h, p); break;
    default: launch_csr_rows<PK_JAC>(h, p); break;
  }
}

void launch_csr(pbicg_ctx* h, Phase p) {
  const CsrOp& A = h->csr;
  // the TMA chunk-ring sweeps apply Jacobi (and block Jacobi b <= 4) themselves
  const bool ring = !h->ilu && h->cst_ok && h->cst_on;
  switch (p) {
    case PH_CCP: {
      LaunchScope ls(h, K_CL1);
      if (ring && h->csr.bj <= 1) c_cl_tma<0><<<h->cst_grid, CST_T, kCstSmem, h->stream>>>(A, h->V, h->scal, h->part, h->hist);
      else launch_rows(h, p);
    } break;
    case PH_SP_CLS: { LaunchScope ls(h, K_SPMVB); launch_spmv<SP_CLS>(h); } break;
    case PH_CCU: {
      LaunchScope ls(h, K_CL2);
      if (ring && h->csr.bj <= 1) c_cl_tma<1><<<h->cst_grid, CST_T, kCstSmem, h->stream>>>(A, h->V, h->scal, h->part, h->hist);
      else launch_rows(h, p);
    } break;
    case PH_SP_CLY: { LaunchScope ls(h, K_SPMVD); launch_spmv<SP_CLY>(h); } break;
    case PH_CCX: {
      LaunchScope ls(h, K_CL3);
      if (h->cst_ok && h->cst_on)  // no M^-1 here: the ring serves every preconditioner
        c_cl_tma<2><<<h->cst_grid, CST_T, kCstSmem, h->stream>>>(A, h->V, h->scal, h->part, h->hist);
      else
        c_cl_x<<<h->grid[K_SWEEPC], h->block, 0, h->stream>>>(A, h->V, h->scal, h->part, h->hist);
    } break;
    case PH_SP_PCW0: { LaunchScope ls(h, K_INIT); launch_spmv<SP_PCW0>(h); } break;
    case PH_SP_PCN: { LaunchScope ls(h, K_SPMVB); launch_spmv<SP_PCN>(h); } break;
    case PH_PRECMV: { LaunchScope ls(h, K_INIT); launch_rows(h, p); } break;
    case PH_CPC: { LaunchScope ls(h, K_PC); launch_rows(h, p); } break;
    case PH_INIT1: {
      LaunchScope ls(h, K_INIT);
      if (h->csr.bj <= 1 && !h->ilu && h->win_ok && !h->auto_rr)  // window SpMV, SELL-32
        c_spmv_win<SP_I1><<<h->win_grid, WNT, WIN_SMEM, h->stream>>>(A, h->V, h->scal, h->wg,
                                                                     h->part, h->hist);
      else launch_rows(h, p);
    } break;
    case PH_INIT2: {
      LaunchScope ls(h, K_INIT);
      if (h->csr.bj <= 1 && !h->ilu && h->win_ok)
        c_spmv_win<SP_I2><<<h->win_grid, WNT, WIN_SMEM, h->stream>>>(A, h->V, h->scal, h->wg,
                                                                     h->part, h->hist);
      else launch_rows(h, p);
    } break;
    case PH_SWEEPA:
    case PH_SWEEPC: {
      const int SW = p == PH_SWEEPA ? 0 : 1;
      LaunchScope ls(h, SW == 0 ? K_SWEEPA : K_SWEEPC);
      if (ring && h->csr.bj <= 4) {  // TMA chunk ring (Jacobi, b <= 4)
        const int g = h->cst_grid;
        const bool bj = h->csr.bj > 1, nrm = h->auto_rr != 0;
#define CST_L(S, N, B) c_sweep_tma<S, N, B><<<g, CST_T, kCstSmem, h->stream>>>(A, h->V, h->scal, h->part, h->hist, 0.0)
        if (SW == 0) {
          if (bj) { if (nrm) CST_L(0, true, true); else CST_L(0, false, true); }
          else { if (nrm) CST_L(0, true, false); else CST_L(0, false, false); }
        } else {
          if (bj) { if (nrm) CST_L(1, true, true); else CST_L(1, false, true); }
          else { if (nrm) CST_L(1, true, false); else CST_L(1, false, false); }
        }
#undef CST_L
      } else {
        launch_rows(h, p);
      }
    } break;
    case PH_SPMVB: {
      LaunchScope ls(h, K_SPMVB);
      if (h->win_ok)
        c_spmv_win<SP_V><<<h->win_grid, WNT, WIN_SMEM, h->stream>>>(A, h->V, h->scal, h->wg,
                                                                    h->part, h->hist);
      else
        c_spmvB<<<h->grid[K_SPMVB], h->block, 0, h->stream>>>(A, h->V, h->scal);
    } break;
    case PH_RR1: { LaunchScope ls(h, K_RR1); launch_rows(h, p); } break;
    case PH_RR2: { LaunchScope ls(h, K_RR2); launch_rows(h, p); } break;
    case PH_SPMVD: {
      LaunchScope ls(h, K_SPMVD);
      if (h->win_ok)
        c_spmv_win<SP_T><<<h->win_grid, WNT, WIN_SMEM, h->stream>>>(A, h->V, h->scal, h->wg,
                                                                    h->part, h->hist);
      else
        c_spmvD<<<h->grid[K_SPMVD], h->block, 0, h->stream>>>(A, h->V, h->scal);
    } break;
    case PH_GAP: {
      LaunchScope ls(h, K_GAP);
      if (h->win_ok)  // window SpMV over the SELL-32 matrix, gap epilogue
        c_spmv_win<SP_GAP><<<h->win_grid, WNT, WIN_SMEM, h->stream>>>(A, h->V, h->scal, h->wg,
                                                                      h->part, h->hist);
      else
        c_gap<<<h->grid[K_GAP], h->block, 0, h->stream>>>(A, h->V, h->scal, h->part, h->hist);
    } break;
    default:
      break;
  }
}

// ILU(0) application out := M^{-1} in (ilu_kernels.cuh; reading A34): forward then
// backward sweep, gated like the step it follows (1: skip when done, 2: only in a
// replacement iteration)
void launch_ilu(pbicg_ctx* h, const double* in, double* out, int gate) {
  LaunchScope ls(h, K_PREC);
  const IluOp& P = h->ilu_op;
  if (h->ilu_st) {
    if (P.dim == 3) {
      k_ilu_st<3, false><<<h->ilu_grid, kIluThreads, kIluSmem, h->stream>>>(P, h->scal, gate, in, out);
      k_ilu_st<3, true><<<h->ilu_grid, kIluThreads, kIluSmem, h->stream>>>(P, h->scal, gate, in, out);
    } else {
      k_ilu_2d<false><<<h->ilu_grid, 32 * I2_W, 0, h->stream>>>(P, h->scal, gate, in, out);
      k_ilu_2d<true><<<h->ilu_grid, 32 * I2_W, 0, h->stream>>>(P, h->scal, gate, in, out);
    }
  } else {
    k_ilu_csr<false><<<h->ilu_grid, 256, 0, h->stream>>>(P, h->scal, gate, in, out);
    k_ilu_csr<true><<<h->ilu_grid, 256, 0, h->stream>>>(P, h->scal, gate, in, out);
  }
}

void launch(pbicg_ctx* h, Phase p) {
  if (h->kind == KIND_CSR) launch_csr(h, p);
  else if (h->dim == 3) launch_stencil<3>(h, p);
  else launch_stencil<2>(h, p);
}

void launch_fin(pbicg_ctx* h, int f) {
  LaunchScope ls(h, K_FIN);
  switch (f) {
    // with automated replacement the reductions also carry the bound norms
    case F_INIT1:
      if (h->auto_rr) k_fin<F_INIT1, 4><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      else k_fin<F_INIT1, 2><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      break;
    case F_INIT2: k_fin<F_INIT2, 1><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_SWEEPA:
      if (h->auto_rr) k_fin<F_SWEEPA, 12><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      else k_fin<F_SWEEPA, 2><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      break;
    case F_SWEEPC:
      if (h->auto_rr) k_fin<F_SWEEPC, 9><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      else k_fin<F_SWEEPC, 5><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      break;
    case F_RR1: k_fin<F_RR1, 4><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_RR2:
      if (h->auto_rr) k_fin<F_RR2, 6><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      else k_fin<F_RR2, 5><<<1, 32, 0, h->stream>>>(h->scal, h->hist);
      break;
    case F_GAP: k_fin<F_GAP, 1><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_CL1: k_fin<F_CL1, 1><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_CL2: k_fin<F_CL2, 2><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_CL3: k_fin<F_CL3, 2><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_PINIT2: k_fin<F_PINIT2, 2><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
    case F_PC: k_fin<F_PC, 3><<<1, 32, 0, h->stream>>>(h->scal, h->hist); break;
  }
}

// ---------------------------------------------------------------------------
// Rank exchange.  Enqueue-only (no host synchronisation); graph-capturable.
using VecSel = std::function<double*(pbicg_ctx*)>;

// exchange the rank rows of the Dot2 partials (exact all-gather: every row but
// the owner's is zero in red_send, so the sum adds exact zeros)
void comm_reduce(const Members& G, bool on_side) {
  pbicg_ctx* h0 = G[0];
  if (!h0->dist) return;
  if (h0->p2p) return;  // the producing kernels already stored into every rank's buffer
  if (h0->comm == COMM_NCCL) {
    pbicg_ctx* h = h0;
    cudaStream_t s = on_side ? h->side : h->stream;
    nccl_api().AllReduce(h->red_send, h->red_recv, (size_t)h->nranks * RED_K * 2, ncclDouble,
                         ncclSum, on_side ? h->nccl_red : h->nccl_halo, s);
  } else {
    cudaStream_t s = on_side ? h0->side : h0->stream;
    for (pbicg_ctx* d : G)
      for (pbicg_ctx* src : G)
        cudaMemcpyAsync(d->red_recv + (size_t)src->rank * RED_K,
                        src->red_send + (size_t)src->rank * RED_K, RED_K * sizeof(Dd),
                        cudaMemcpyDeviceToDevice, s);
  }
}

// Stencil schedule in force: 2 = the paper's split 4-phase schedule, else the fused
// 2-sweep one.  schedule 0 (auto) picks split for NCCL ranks whose slab is small
// enough that the two reductions the fused schedule can hide only behind a halo
// exchange cost more than the split schedule's 8 extra passes (DESIGN.md section 2:
// n_local < 2 t_red BW / 64 B = 3 M rows at t_red = 15 us, 6.5 TB/s -- a model, the
// 1-GPU pool cannot measure it); never with the peer-memory transport (a few-us
// reduction), block Jacobi, automated replacement or the comparison methods.
bool split_sched(const pbicg_ctx* h) {
  if (h->kind != KIND_STENCIL) return false;
  if (h->schedule == 2) return true;
  return h->schedule == 0 && h->auto_split && !h->p2p && h->method == M_PBICGSTAB &&
         !h->auto_rr && h->tg.bj <= 1;
}

// the stencil replacement step runs on the tile kernels: RR2 forms w = A k, z = A l from
// the stored k, l (their ghost planes move instead of r, s; tile_sweeps.cuh Stash)
bool tile_rr(const pbicg_ctx* h) {
  return h->kind == KIND_STENCIL && h->tile_ok && (h->tile_on || h->auto_rr);
}

// the fused schedule's z / w halos travel inside the tile sweeps (transport 1)
bool fused_halo(const pbicg_ctx* h) {
  return h->p2p && h->kind == KIND_STENCIL && h->tile_ok && h->tile_on && !split_sched(h);
}

// nearest-neighbour ghost exchange of halo_n rows per side for each vector
void comm_halo(const Members& G, std::initializer_list<VecSel> sels) {
  pbicg_ctx* h0 = G[0];
  if (!h0->dist) return;
  h0->halo_ops++;
  if (h0->comm == COMM_NCCL) {
    pbicg_ctx* h = h0;
    auto& api = nccl_api();
    api.GroupStart();
    for (auto& sel : sels) {
      double* v = sel(h);
      if (h->rank > 0) {
        api.Send(v, h->halo_n, ncclDouble, h->rank - 1, h->nccl_halo, h->stream);
        api.Recv(v - h->halo_n, h->halo_n, ncclDouble, h->rank - 1, h->nccl_halo, h->stream);
      }
      if (h->rank < h->nranks - 1) {
        api.Send(v + h->n_local - h->halo_n, h->halo_n, ncclDouble, h->rank + 1, h->nccl_halo,
                 h->stream);
        api.Recv(v + h->n_local, h->halo_n, ncclDouble, h->rank + 1, h->nccl_halo, h->stream);
      }
    }
    api.GroupEnd();
  } else {
    const size_t nb = (size_t)h0->halo_n * sizeof(double);
    for (auto& sel : sels) {
      for (size_t r = 0; r < G.size(); ++r) {
        pbicg_ctx* me = G[r];
        double* v = sel(me);
        if (r > 0) {  // my first rows -> left neighbour's upper ghost
          pbicg_ctx* nbr = G[r - 1];
          cudaMemcpyAsync(sel(nbr) + nbr->n_local, v, nb, cudaMemcpyDeviceToDevice, h0->stream);
        }
        if (r + 1 < G.size()) {  // my last rows -> right neighbour's lower ghost
          pbicg_ctx* nbr = G[r + 1];
          cudaMemcpyAsync(sel(nbr) - nbr->halo_n, v + me->n_local - me->halo_n, nb,
                          cudaMemcpyDeviceToDevice, h0->stream);
        }
      }
    }
  }
}

// reduction on the side stream, ordered after everything enqueued so far
void fork_reduce(const Members& G) {
  pbicg_ctx* h0 = G[0];
  cudaEventRecord(h0->ev_fork, h0->stream);
  cudaStreamWaitEvent(h0->side, h0->ev_fork, 0);
  comm_reduce(G, true);
  cudaEventRecord(h0->ev_join, h0->side);
}
void join_reduce(const Members& G) { cudaStreamWaitEvent(G[0]->stream, G[0]->ev_join, 0); }

void each(const Members& G, Phase p) {
  for (pbicg_ctx* h : G) launch(h, p);
}
// ILU(0) handles: out := M^{-1} in on every member (each rank its own block, A34);
// a no-op for the point-wise preconditioners, which the kernels apply themselves
void each_ilu(const Members& G, const VecSel& in, const VecSel& out, int gate) {
  if (!G[0]->ilu) return;
  for (pbicg_ctx* h : G) launch_ilu(h, in(h), out(h), gate);
}
void each_fin(const Members& G, int f) {
  if (!G[0]->dist) return;
  for (pbicg_ctx* h : G) launch_fin(h, f);
}
void reduce_fin(const Members& G, int f) {
  if (!G[0]->dist) return;
  comm_reduce(G, false);
  each_fin(G, f);
}

const VecSel SX = [](pbicg_ctx* h) { return h->V.x; };
const VecSel SG = [](pbicg_ctx* h) { return h->V.g; };
const VecSel SR = [](pbicg_ctx* h) { return h->V.r; };
const VecSel SS = [](pbicg_ctx* h) { return h->V.s; };
const VecSel SW0 = [](pbicg_ctx* h) { return h->V.w0; };
const VecSel SW1 = [](pbicg_ctx* h) { return h->V.w1; };
const VecSel SZ0 = [](pbicg_ctx* h) { return h->V.z0; };
const VecSel SZ1 = [](pbicg_ctx* h) { return h->V.z1; };
const VecSel SNV = [](pbicg_ctx* h) { return h->V.nv; };
const VecSel SMV = [](pbicg_ctx* h) { return h->V.mv; };
const VecSel SK = [](pbicg_ctx* h) { return h->V.k; };
const VecSel SL = [](pbicg_ctx* h) { return h->V.l; };
const VecSel SZRR = [](pbicg_ctx* h) { return h->V.zrr; };

// Alg. 1 (method 1) on the stencil: p_i, s_i, r_i double-buffered by parity
// (tile_sweeps.cuh TM_CL*): r in {r, k}, p in {g, l}, s in {s, zrr}
// CSR: p in g, M^-1 p in mv, M^-1 q in nv, y in z1 (csr_kernels.cuh c_cl_*)
const VecSel SNVv = [](pbicg_ctx* h) { return h->V.nv; };
const VecSel SMVv = [](pbicg_ctx* h) { return h->V.mv; };

void enq_iter_classic_csr(const Members& G) {
  const bool dist = G[0]->dist;
  each(G, PH_CCP);  // l.17 (previous i) + l.4: p_i, M^-1 p_i
  each_ilu(G, SG, SMVv, 1);  // ILU(0): M^-1 p_i
  if (dist) comm_halo(G, {SMVv});
  each(G, PH_SP_CLS);  // l.5-6: s_i, (r^0, s_i) -> alpha
  reduce_fin(G, F_CL1);
  each(G, PH_CCU);  // l.8-9: u = M^-1 (r - alpha s)
  each_ilu(G, SZ0, SNVv, 1);  // ILU(0): q_i was stored in z0
  if (dist) comm_halo(G, {SNVv});
  each(G, PH_SP_CLY);  // l.10-11: y, (q,y), (y,y) -> omega
  reduce_fin(G, F_CL2);
  each(G, PH_CCX);  // l.13-16: x, r, (r^0,r), ||r|| -> beta
  reduce_fin(G, F_CL3);
}

// p-CG on CSR, software-pipelined: iteration i enqueues the SpMV of iteration
// i+1 (n_{i+1} = A m_{i+1}) between its reduction's fork and join, so on P ranks
// the all-reduce of {(r,u),(w,u),||r||} overlaps that SpMV -- the point of p-CG
void enq_iter_pipecg_csr(const Members& G) {
  pbicg_ctx* h0 = G[0];
  const bool dist = h0->dist;
  each(G, PH_CPC);
  if (!dist) {
    each_ilu(G, SW0, SMVv, 1);  // ILU(0): m_{i+1} = M^-1 w_{i+1}
    each(G, PH_SP_PCN);
    return;
  }
  if (h0->overlap) fork_reduce(G);
  else comm_reduce(G, false);
  each_ilu(G, SW0, SMVv, 1);  // overlaps the reduction with the SpMV
  comm_halo(G, {SMVv});
  each(G, PH_SP_PCN);
  if (h0->overlap) join_reduce(G);
  each_fin(G, F_PC);
}

void enq_init_classic(const Members& G) {
  const bool dist = G[0]->dist;
  if (dist) comm_halo(G, {SX});
  each(G, PH_INIT1);  // r0 := b - A x0, r^0 := r0; rho_0, ||b|| (F_INIT1, method 1)
  reduce_fin(G, F_INIT1);
  if (dist) comm_halo(G, {SR});
}

void enq_iter_classic(const Members& G, int par) {
  const bool dist = G[0]->dist;
  each(G, PH_CL1);  // l.17 (previous i) + l.4-6: p_i, s_i, (r^0, s_i)
  if (dist) {
    comm_reduce(G, false);
    comm_halo(G, {par ? SL : SG, par ? SZRR : SS});  // p_i, s_i ghosts
    each_fin(G, F_CL1);
  }
  each(G, PH_CL2);  // l.8-12: (q, y), (y, y) -> omega
  reduce_fin(G, F_CL2);
  each(G, PH_CL3);  // l.13-16: x, r; (r^0, r), ||r|| -> beta
  reduce_fin(G, F_CL3);
  if (dist) comm_halo(G, {par ? SR : SK});  // r_{i+1}
}

// p-CG (method 2): one kernel and one reduction per iteration
void enq_init_pipecg(const Members& G) {
  const bool dist = G[0]->dist;
  if (G[0]->kind == KIND_CSR) {
    if (dist) comm_halo(G, {SX});
    each(G, PH_INIT1);  // r0, u0 (k); ||r0||, ||b|| (F_INIT1, method 2)
    each_ilu(G, SR, SK, 0);  // ILU(0): u0 = M^-1 r0
    reduce_fin(G, F_INIT1);
    if (dist) comm_halo(G, {SK});
    each(G, PH_SP_PCW0);  // w0 = A u0; (r0,u0), (w0,u0) -> alpha_0
    reduce_fin(G, F_PINIT2);
    if (G[0]->ilu) each_ilu(G, SW0, SMVv, 0);
    else each(G, PH_PRECMV);   // m0 = M^-1 w0
    if (dist) comm_halo(G, {SMVv});
    each(G, PH_SP_PCN);  // n_0 = A m_0
    return;
  }
  if (dist) comm_halo(G, {SX});
  each(G, PH_PCI1);  // r0, u0; ||r0||, ||b|| (F_INIT1, method 2)
  reduce_fin(G, F_INIT1);
  if (dist) comm_halo(G, {SR});
  each(G, PH_PCI2);  // w0 = A u0; (r0,u0), (w0,u0) -> alpha_0
  reduce_fin(G, F_PINIT2);
  if (dist) comm_halo(G, {SW0});
}

void enq_iter_pipecg(const Members& G, int par) {
  const bool dist = G[0]->dist;
  each(G, PH_PC);
  reduce_fin(G, F_PC);
  if (dist) comm_halo(G, {par ? SW0 : SW1});  // w_{i+1}
}

void enq_gap(const Members& G) {
  if (!G[0]->gap_on) return;
  if (G[0]->dist) comm_halo(G, {SX});
  each(G, PH_GAP);
  reduce_fin(G, F_GAP);
}

// Alg. 2 lines 2-3 [+ gap of iteration 0]
void enq_init(const Members& G) {
  pbicg_ctx* h0 = G[0];
  const bool dist = h0->dist;
  if (h0->method != M_PBICGSTAB) {
    if (h0->method == M_BICGSTAB) enq_init_classic(G);
    else enq_init_pipecg(G);
    enq_gap(G);
    return;
  }
  if (dist) comm_halo(G, {SX});
  each(G, PH_INIT1);
  each_ilu(G, SR, SK, 0);  // ILU(0): k0 = M^-1 r0
  reduce_fin(G, F_INIT1);
  if (dist) comm_halo(G, {h0->kind == KIND_CSR ? SK : SR});  // CSR: w0 = A k0
  each(G, PH_INIT2);
  each_ilu(G, SW0, SMV, 0);  // ILU(0): m0 = M^-1 w0
  reduce_fin(G, F_INIT2);
  if (h0->kind == KIND_CSR) {  // t_0 = A m_0 (line 3)
    if (dist) comm_halo(G, {SMV});
    each(G, PH_SPMVD);
  } else {
    if (dist) comm_halo(G, {SW0});  // w_0 is read with the stencil
    if (split_sched(h0)) each(G, PH_SPD);  // split schedule: t_0 stored
  }
  if (h0->gap_on) {
    each(G, PH_GAP);
    reduce_fin(G, F_GAP);
  }
}

// one iteration i (par = i & 1 selects the double-buffered w and z)
void enq_iter(const Members& G, bool with_rr, int par) {
  pbicg_ctx* h0 = G[0];
  const bool dist = h0->dist;
  if (h0->method != M_PBICGSTAB) {
    if (h0->kind == KIND_CSR) {
      if (h0->method == M_BICGSTAB) enq_iter_classic_csr(G);
      else enq_iter_pipecg_csr(G);
    } else if (h0->method == M_BICGSTAB) {
      enq_iter_classic(G, par);
    } else {
      enq_iter_pipecg(G, par);
    }
    enq_gap(G);
    return;
  }
  if (split_sched(h0)) {
    // split 4-phase schedule (the paper's): each reduction hides behind the
    // halo exchange + stand-alone SpMV of the vector the next phase needs
    const bool ov = dist && h0->overlap;
    each(G, PH_SWEEPA2);  // lines 5-12 with stored t_i, v_{i-1}
    if (ov) fork_reduce(G);
    else if (dist) comm_reduce(G, false);
    if (dist) comm_halo(G, {par ? SZ1 : SZ0});
    each(G, PH_SPB);  // lines 13-14: v_i = A M^-1 z_i
    if (ov) join_reduce(G);
    each_fin(G, F_SWEEPA);
    each(G, PH_SWEEPC2);  // lines 16-21
    if (ov && !with_rr) {  // reduction #2 || halo w_{i+1} + SpMV_D (no replacement possible)
      fork_reduce(G);
      comm_halo(G, {par ? SW0 : SW1});
      each(G, PH_SPD);  // lines 22-23 (harmless if this iteration converged)
      join_reduce(G);
      each_fin(G, F_SWEEPC);
    } else {
      reduce_fin(G, F_SWEEPC);
      if (with_rr) {  // eq:rr after line 20
        if (dist) comm_halo(G, {SX, SG});
        each(G, PH_RR1);
        if (h0->auto_rr) reduce_fin(G, F_RR1);
        if (dist) {
          if (tile_rr(h0)) comm_halo(G, {SK, SL});
          else comm_halo(G, {SR, SS});
        }
        each(G, PH_RR2);
        reduce_fin(G, F_RR2);
      }
      if (dist) comm_halo(G, {par ? SW0 : SW1});
      each(G, PH_SPD);  // t_{i+1} from the (replaced) w_{i+1} (A27)
    }
    if (h0->gap_on) {
      if (dist) comm_halo(G, {SX});
      each(G, PH_GAP);
      reduce_fin(G, F_GAP);
    }
    return;
  }
  if (h0->kind == KIND_STENCIL) {
    // fused 2-sweep schedule: sweep A (l.5-12) -> omega; sweep C (l.16-21) -> beta, alpha.
    // P ranks: each reduction runs on the side stream (own communicator) while the
    // halo of the vector the next sweep reads with its stencil moves on the compute
    // stream (the exchange the reduction can hide behind)
    each(G, PH_SWEEPA);
    if (dist) {
      const bool ov = h0->overlap != 0;
      if (ov) {
        fork_reduce(G);
      } else {
        comm_reduce(G, false);
      }
      // z_i for sweep C's stencil (transport 1: sweep A stored it in the neighbours)
      if (!fused_halo(h0)) comm_halo(G, {par ? SZ1 : SZ0});
      if (ov) join_reduce(G);
      each_fin(G, F_SWEEPA);
    }
    each(G, PH_SWEEPC);
    if (dist && !with_rr && h0->overlap) {
      // reduction #2 || halo of w_{i+1} (no replacement can rewrite w this iteration)
      fork_reduce(G);
      if (!fused_halo(h0)) comm_halo(G, {par ? SW0 : SW1});
      join_reduce(G);
      each_fin(G, F_SWEEPC);
      if (h0->gap_on) {
        comm_halo(G, {SX});
        each(G, PH_GAP);
        reduce_fin(G, F_GAP);
      }
      return;
    }
    reduce_fin(G, F_SWEEPC);
    if (with_rr) {  // eq:rr after line 20
      if (dist) comm_halo(G, {SX, SG});
      each(G, PH_RR1);
      if (h0->auto_rr) reduce_fin(G, F_RR1);  // norms of the replaced vectors
      if (dist) {
        if (tile_rr(h0)) comm_halo(G, {SK, SL});
        else comm_halo(G, {SR, SS});
      }
      each(G, PH_RR2);
      reduce_fin(G, F_RR2);
    }
    // w_{i+1} (transport 1: stored by sweep C in the neighbours unless replaced)
    if (dist && (with_rr || !fused_halo(h0))) comm_halo(G, {par ? SW0 : SW1});
  } else {
    // split 4-phase schedule: reduction #1 overlaps M^-1 z (ILU(0)), the halo
    // and spmv_B; reduction #2 overlaps M^-1 w, the halo and spmv_D when this
    // iteration cannot replace
    each(G, PH_SWEEPA);
    const bool ov = dist && h0->overlap;
    if (ov) fork_reduce(G);
    else if (dist) comm_reduce(G, false);
    each_ilu(G, SZ0, SNV, 1);  // ILU(0): n_i = M^-1 z_i (line 13)
    if (dist) comm_halo(G, {SNV});  // n_i ghosts for v_i = A n_i
    each(G, PH_SPMVB);  // lines 13-14
    if (ov) join_reduce(G);
    each_fin(G, F_SWEEPA);
    each(G, PH_SWEEPC);
    if (ov && !with_rr) {
      fork_reduce(G);
      each_ilu(G, SW0, SMV, 1);  // ILU(0): m_{i+1} = M^-1 w_{i+1} (line 22)
      comm_halo(G, {SMV});
      each(G, PH_SPMVD);  // lines 22-23 (harmless if this iteration converged)
      join_reduce(G);
      each_fin(G, F_SWEEPC);
    } else {
      reduce_fin(G, F_SWEEPC);
      if (with_rr) {
        if (dist) comm_halo(G, {SX, SG});
        each(G, PH_RR1);
        each_ilu(G, SR, SK, 2);  // ILU(0): k := M^-1 r, l := M^-1 s (eq:rr)
        each_ilu(G, SS, SL, 2);
        if (h0->auto_rr) reduce_fin(G, F_RR1);  // norms of the replaced vectors
        if (dist) comm_halo(G, {SK, SL});         // w := A k, z := A l
        each(G, PH_RR2);
        reduce_fin(G, F_RR2);
      }
      each_ilu(G, SW0, SMV, 1);  // ILU(0): m_{i+1} from the (replaced) w (A27)
      if (dist) comm_halo(G, {SMV});  // m_{i+1} ghosts
      each(G, PH_SPMVD);  // lines 22-23
    }
  }
  if (h0->gap_on) {
    if (dist) comm_halo(G, {SX});
    each(G, PH_GAP);
    reduce_fin(G, F_GAP);
  }
}

// chunk of L iterations starting at a multiple of L (L even, multiple of P when
// P > 0): offset o replaces iff P > 0 && (o+1) % P == 0.
void enq_chunk(const Members& G, int L, int P) {
  // automated replacement: decided on the device, so every iteration carries the
  // (early-exiting) replacement kernels
  const bool every = G[0]->auto_rr != 0;
  for (int o = 0; o < L; ++o) {
    const bool rr = every || (P > 0 && ((o + 1) % P) == 0);
    enq_iter(G, rr, o & 1);
  }
}

void destroy_graphs(pbicg_ctx* h) {
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
}

pbicg_status run_chunk(const Members& G, int L, int P) {
  pbicg_ctx* h = G[0];
  const bool graphs = h->use_graphs && !h->timing;
  if (!graphs) {
    enq_chunk(G, L, P);
    CU(cudaGetLastError());
    return PBICG_OK;
  }
  std::vector<std::vector<int64_t>> before;
  for (pbicg_ctx* m : G) before.emplace_back(m->launches, m->launches + K_N);
  auto key = std::make_tuple(L, P, h->gap_on * 2 + h->auto_rr);
  auto it = h->graphs.find(key);
  // the enqueue pass below (capture or, for cached graphs, counted separately)
  // establishes how many launches one replay contains
  // A capture that fails (e.g. a communication library that cannot be captured on
  // this system) is not fatal: the handle's members drop to direct enqueue, which is
  // the same sequence of launches, and this chunk runs that way.
  auto no_graphs = [&](cudaGraph_t g) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    for (size_t q = 0; q < G.size(); ++q) {  // the failed capture counted its launches
      G[q]->use_graphs = 0;
      for (int k = 0; k < K_N; ++k) G[q]->launches[k] = before[q][k];
    }
    enq_chunk(G, L, P);
    CU(cudaGetLastError());
    return PBICG_OK;
  };
  if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return no_graphs(nullptr);
  enq_chunk(G, L, P);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
  if (ce != cudaSuccess) return no_graphs(g);
  if (it == h->graphs.end()) {
    cudaGraphExec_t ge = nullptr;
    ce = cudaGraphInstantiate(&ge, g, 0);
    if (ce != cudaSuccess) return no_graphs(g);
    it = h->graphs.emplace(key, ge).first;
  }
  cudaGraphDestroy(g);
  CU(cudaGraphLaunch(it->second, h->stream));
  return PBICG_OK;
}

pbicg_status ensure_hist(pbicg_ctx* h, int64_t need) {
  if (need <= h->hist_cap) return PBICG_OK;
  destroy_graphs(h);  // graphs captured the old pointers
  int64_t cap = need < 1024 ? 1024 : need;
  void *a = nullptr, *b = nullptr, *c = nullptr, *d = nullptr, *e = nullptr;
  ST(dalloc(h, &a, (size_t)cap * sizeof(double)));
  ST(dalloc(h, &b, (size_t)cap * sizeof(double)));
  ST(dalloc(h, &c, (size_t)cap * sizeof(double)));
  ST(dalloc(h, &d, (size_t)cap * sizeof(int32_t)));
  ST(dalloc(h, &e, (size_t)cap * SC_W * sizeof(double)));
  h->hist.rnorm = (double*)a;
  h->hist.gap = (double*)b;
  h->hist.fr = (double*)c;
  h->hist.rrl = (int32_t*)d;
  h->hist.sc = (double*)e;
  h->hist_cap = cap;
  return PBICG_OK;
}

template <int DIM, int MODE>
cudaError_t set_tile_attr(pbicg_ctx* h) {
  const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if (h->tile_seg) {
    int occ = 1;
    const cudaError_t e = tile_seg_attr(DIM, MODE, (int)h->tile_smem[MODE], &occ);
    h->tile_occ[MODE] = occ < 1 ? 1 : occ;
    return e;
  }
  // light modes (few streams) fit 2 CTAs per SM: twice the bytes in flight
  int occ = 1, occ0 = 1;
  cudaError_t e = tile_jac_attr_1(DIM, MODE, (int)h->tile_smem[MODE], &occ);
  if (e == cudaSuccess) e = tile_jac_attr_0(DIM, MODE, (int)h->tile_smem[MODE], &occ0);
  (void)A;
  if constexpr (bj_mode(MODE)) {
    if (e == cudaSuccess && h->tg.bj > 1) {
      const int sm = (int)h->tile_smem[MODE];
      if (h->tg.bj == 2) e = tile_bj_attr_2(DIM, MODE, sm, &occ);
      else if (h->tg.bj == 4) e = tile_bj_attr_4(DIM, MODE, sm, &occ);
      else e = tile_bj_attr_8(DIM, MODE, sm, &occ);
    }
  }
  h->tile_occ[MODE] = occ < 1 ? 1 : occ;
  return e;
}

template <int DIM>
cudaError_t set_tile_attrs(pbicg_ctx* h) {
  cudaError_t e = set_tile_attr<DIM, TM_A>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_C>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_RR1>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_RR2>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_GAP>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_INIT1>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_INIT2>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_CL1>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_CL2>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_CL3>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_PC>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_PCI1>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_PCI2>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_AN>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_CN>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_RR1N>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_RR2N>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_INIT1N>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_SPB>(h);
  if (e == cudaSuccess) e = set_tile_attr<DIM, TM_SPD>(h);
  return e;
}

// Tall tiles of the light steps (spmv_tile.cuh): TY lines with NP row pairs per thread
// (LtTraits), chunks of planes as for the sweeps.  The SpMVs and the replacement step
// have their own geometry; RR1 and RR2 share theirs (the dot stash is per CTA).
template <int MODE>
cudaError_t light_attr(size_t smem) {
  return cudaFuncSetAttribute(t_light3<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem);
}

// lines per tile and chunking for NP row pairs per thread; false if nothing fits
bool light_geo(const pbicg_ctx* h, int np, int smem_cap, size_t (*smem)(const SpmvGeo&),
               SpmvGeo& q) {
  const Geo& g = h->geo;
  int64_t TY = (2LL * TNT * np) / g.nx;
  if (TY > g.ny) TY = g.ny;
  for (; TY >= 1; --TY) {
    q.TY = (int32_t)TY;
    q.sv_stride = (int32_t)((TY * g.nx + 2 * (g.nx + 2) + 2 + 1) & ~1LL);
    q.st_stride = (int32_t)((TY * g.nx + 2 + 1) & ~1LL);
    if (smem(q) <= (size_t)smem_cap) break;
  }
  if (TY < 1) return false;
  q.ncols = (int32_t)((g.ny + TY - 1) / TY);
  const int grid = h->num_sm;
  int64_t best_n = 1;
  double best_w = 1e30;
  for (int64_t nch = 1; nch <= g.nol; ++nch) {
    const int64_t chunk = (g.nol + nch - 1) / nch;
    const int64_t nchk = (g.nol + chunk - 1) / chunk;
    const int64_t units = nchk * q.ncols;
    const int64_t rounds = (units + grid - 1) / grid;
    const double w = (double)rounds * (double)(chunk + 2);
    if (w < best_w - 1e-9) {
      best_w = w;
      best_n = nch;
    }
    if (units > 64LL * grid) break;
  }
  q.chunk = (int32_t)((g.nol + best_n - 1) / best_n);
  q.units = (int32_t)(((g.nol + q.chunk - 1) / q.chunk) * q.ncols);
  return true;
}

size_t smem_spmv(const SpmvGeo& q) { return light_smem_bytes<TM_SPB>(q); }
size_t smem_rr(const SpmvGeo& q) {
  const size_t a = light_smem_bytes<TM_RR1>(q), b = light_smem_bytes<TM_RR2>(q);
  return a > b ? a : b;
}

void setup_light_tiles(pbicg_ctx* h, int smem_cap) {
  h->spt_ok = h->lrr_ok = false;
  if (h->dim != 3 || !h->tile_ok || h->tile_seg || !h->tile_vec || h->tg.bj > 1) return;
  const char* off = getenv("PBICG_LIGHT");  // tuning experiments only: 0 = t_tile everywhere
  if (off && strtol(off, nullptr, 10) == 0) return;
  if (light_geo(h, LtTraits<TM_SPB>::NP, smem_cap, smem_spmv, h->sq)) {
    h->spt_smem = smem_spmv(h->sq);
    if (light_attr<TM_SPB>(h->spt_smem) == cudaSuccess &&
        light_attr<TM_SPD>(h->spt_smem) == cudaSuccess)
      h->spt_ok = true;
  }
  if (light_geo(h, LtTraits<TM_RR1>::NP, smem_cap, smem_rr, h->sq_rr)) {
    h->lrr_smem = smem_rr(h->sq_rr);
    if (light_attr<TM_RR1>(h->lrr_smem) == cudaSuccess &&
        light_attr<TM_RR2>(h->lrr_smem) == cudaSuccess)
      h->lrr_ok = true;
  }
  cudaGetLastError();
}

template <int MODE>
void launch_light(pbicg_ctx* h) {
  const bool rr = MODE == TM_RR1 || MODE == TM_RR2;
  const SpmvGeo& q = rr ? h->sq_rr : h->sq;
  const int grid = q.units < h->num_sm ? q.units : h->num_sm;  // RR1, RR2: the same grid
  t_light3<MODE><<<grid, TNT, rr ? h->lrr_smem : h->spt_smem, h->stream>>>(
      h->tg, q, h->V, h->scal, h->part, h->hist);
}

// Tile geometry of the TMA 2.5D sweeps (tile_sweeps.cuh): TY full x-lines per
// tile (3D) or one x-line (2D), a chunk of planes per work unit, units spread
// statically over one CTA per SM (deterministic accumulation order).
void setup_tile(pbicg_ctx* h) {
  const Geo& g = h->geo;
  TileGeo& t = h->tg;
  h->tile_ok = false;
  h->tile_seg = false;
  const int dim = h->dim;
  const int64_t tpmax = 2LL * TNT;  // one row pair per thread
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
  const size_t reserve = 8192;  // static shared memory of the block reductions (K <= 16 pairs)
  const int64_t lines = dim == 3 ? g.ny : 1;
  t.nx = g.nx;
  t.ny = lines;
  t.nol = g.nol;
  t.o0 = g.o0;
  t.nog = g.nog;
  t.pxy = g.pxy;
  t.sx = (int32_t)g.nx;
  t.nseg = 1;
  t.lstride = (int32_t)g.nx;
  int64_t nseg = 1;
  // full-line tiles need nx <= 2 TNT and (3D) a plane of TY >= 1 lines plus two halo
  // lines per staged vector in shared memory (3D: nx <= ~850 for the widest mode, sweep A)
  bool full = g.nx <= tpmax;
  const char* force_seg = getenv("PBICG_TILE_SEG");  // tuning experiments only: x-segment width
  if (force_seg && g.nx % 2 == 0) full = false;
  if (full) {
    int64_t TY = dim == 3 ? (tpmax / g.nx) : 1;
    if (TY > lines) TY = lines;
    t.TY = (int32_t)(TY < 1 ? 1 : TY);
    for (; t.TY >= 1; --t.TY) {
      const int64_t TP = t.TY * g.nx, hl = dim == 3 ? g.nx + 2 : 2;
      t.st_stride = (int32_t)((TP + 2 + 1) & ~1LL);
      t.sv_stride = (int32_t)((TP + 2 * hl + 2 + 1) & ~1LL);
      size_t worst = 0;
      for (int m = 0; m < TM_N; ++m)
        worst = tile_smem_bytes(t, m) > worst ? tile_smem_bytes(t, m) : worst;
      if (worst + reserve <= (size_t)max_smem) break;
    }
    full = t.TY >= 1;
  }
  if (!full) {
    // x-segmented tiles (tile_seg.cu): TY lines x sx columns, sx the widest multiple of
    // 16 (<= 512) whose worst-mode shared memory fits; odd nx keeps the line kernels
    if (g.nx % 2 != 0) return;
    const int64_t TYs = dim == 3 ? (lines < 2 ? lines : 2) : 1;
    int64_t SX = 512;
    if (force_seg) {
      const long v = strtol(force_seg, nullptr, 10);
      if (v >= 64 && v <= 512 && v % 16 == 0) SX = v;
    }
    for (; SX >= 64; SX -= 16) {
      t.TY = (int32_t)TYs;
      t.sx = (int32_t)SX;
      t.lstride = (int32_t)(SX + 2 * SEG_HX);
      t.halo = 0;
      t.st_stride = (int32_t)(TYs * SX);
      t.sv_stride = (int32_t)((dim == 3 ? TYs + 2 : 1) * t.lstride + 2);
      size_t worst = 0;
      for (int m = 0; m < TM_N; ++m)
        worst = tile_smem_bytes(t, m) > worst ? tile_smem_bytes(t, m) : worst;
      if (worst + reserve <= (size_t)max_smem) break;
    }
    if (SX < 64) return;
    nseg = (g.nx + SX - 1) / SX;
    t.nseg = (int32_t)nseg;
    h->tile_seg = true;
    h->tile_vec = true;
    for (int i = 0; i < 7; ++i) t.c[i] = g.c[i];
    t.dinv = g.dinv;
    t.ncols = (int32_t)(((lines + TYs - 1) / TYs) * nseg);
  }
  if (!h->tile_seg) {  // full-line tiles: TY lines of nx
    int64_t TY = dim == 3 ? (tpmax / g.nx) : 1;
    if (TY < 1) TY = 1;
    if (TY > lines) TY = lines;
    if (const char* e = getenv("PBICG_TILE_TY")) {  // tuning experiments only
      const long v = strtol(e, nullptr, 10);
      if (v >= 1 && v < TY) TY = v;
    }
    h->tile_vec = (g.nx % 2) == 0;  // 16-byte aligned pairs / ranges
    for (; TY >= 1; --TY) {
      t.TY = (int32_t)TY;
      t.halo = (int32_t)(dim == 3 ? g.nx + 2 : 2);
      const int64_t TP = TY * g.nx;
      t.st_stride = (int32_t)((TP + 2 + 1) & ~1LL);
      t.sv_stride = (int32_t)((TP + 2 * t.halo + 2 + 1) & ~1LL);
      size_t worst = 0;
      for (int m = 0; m < TM_N; ++m)
        worst = tile_smem_bytes(t, m) > worst ? tile_smem_bytes(t, m) : worst;
      if (worst + reserve <= (size_t)max_smem) break;
    }
    if (TY < 1) return;
    for (int i = 0; i < 7; ++i) t.c[i] = g.c[i];
    t.dinv = g.dinv;
    t.ncols = (int32_t)((lines + TY - 1) / TY);
  }
  // chunk count: minimise rounds * (chunk + 2 prologue planes) per CTA
  const int grid = h->num_sm;
  int64_t best_n = 1;
  double best_w = 1e30;
  for (int64_t nch = 1; nch <= g.nol; ++nch) {
    const int64_t chunk = (g.nol + nch - 1) / nch;
    const int64_t nchk = (g.nol + chunk - 1) / chunk;
    const int64_t units = nchk * t.ncols;
    const int64_t rounds = (units + grid - 1) / grid;
    const double w = (double)rounds * (double)(chunk + 2);
    if (w < best_w - 1e-9) {
      best_w = w;
      best_n = nch;
    }
    if (units > 64LL * grid) break;
  }
  if (const char* e = getenv("PBICG_TILE_NCHUNKS")) {  // tuning experiments only
    const long v = strtol(e, nullptr, 10);
    if (v >= 1 && v <= g.nol) best_n = v;
  }
  t.chunk = (int32_t)((g.nol + best_n - 1) / best_n);
  t.nchunks = (int32_t)((g.nol + t.chunk - 1) / t.chunk);
  t.units = t.nchunks * t.ncols;
  for (int m = 0; m < TM_N; ++m) h->tile_smem[m] = tile_smem_bytes(t, m);
  const cudaError_t e = dim == 3 ? set_tile_attrs<3>(h) : set_tile_attrs<2>(h);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  h->tile_ok = true;
  setup_light_tiles(h, max_smem - (int)reserve);
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
  int prio_lo = 0, prio_hi = 0;  // the reduction side stream: highest priority
  CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, prio_hi));
  CU(cudaEventCreateWithFlags(&h->ev_entry, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_poll[0], cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_poll[1], cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  void* p = nullptr;
  ST(dalloc(h, &p, sizeof(Scal)));
  h->scal = (Scal*)p;
  CU(cudaMemsetAsync(h->scal, 0, sizeof(Scal), h->stream));
  CU(cudaMallocHost(&h->scal_host, 2 * sizeof(Scal)));
  return PBICG_OK;
}

pbicg_status alloc_common(pbicg_ctx* h) {
  double** vs[] = {&h->V.x, &h->V.r, &h->V.rh, &h->V.k, &h->V.g, &h->V.s, &h->V.l, &h->V.b,
                   &h->V.w0, &h->V.w1, &h->V.z0, &h->V.z1, &h->V.zrr, &h->xtmp};
  for (double** v : vs) ST(gvec(h, v));
  const int nr = h->nranks;
  void *a = nullptr, *b = nullptr;
  ST(dalloc(h, &a, (size_t)nr * RED_K * sizeof(Dd)));
  ST(dalloc(h, &b, (size_t)nr * RED_K * sizeof(Dd)));
  h->red_send = (Dd*)a;
  h->red_recv = (Dd*)b;
  CU(cudaMemsetAsync(a, 0, (size_t)nr * RED_K * sizeof(Dd), h->stream));
  CU(cudaMemsetAsync(b, 0, (size_t)nr * RED_K * sizeof(Dd), h->stream));
  int gmax = h->num_sm;
  for (int k = 0; k < K_N; ++k) gmax = h->grid[k] > gmax ? h->grid[k] : gmax;
  void* p = nullptr;
  ST(dalloc(h, &p, (size_t)gmax * RED_K * sizeof(Dd)));  // K <= RED_K partials per CTA
  h->part = (Dd*)p;
  void* q = nullptr;  // the tile replacement step's per-CTA dot stash (tile_sweeps.cuh)
  ST(dalloc(h, &q, (size_t)gmax * STASH_K * sizeof(Dd)));
  h->V.stash = (Dd*)q;
  ST(ensure_hist(h, 1024));
  // rank fields of the device state (kept across solves)
  Scal s;
  memset(&s, 0, sizeof(s));
  s.nranks = h->nranks;
  s.rank = h->rank;
  s.dist = h->dist;
  s.red_send = h->red_send;
  s.red_recv = h->red_recv;
  CU(cudaMemcpyAsync(h->scal, &s, sizeof(Scal), cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return PBICG_OK;
}

// order the handle's stream after prior work on the legacy default stream
pbicg_status entry_sync(pbicg_ctx* h) {
  if (h->own_stream || h->comm == COMM_LOOP) {
    CU(cudaEventRecord(h->ev_entry, 0));
    CU(cudaStreamWaitEvent(h->stream, h->ev_entry, 0));
  }
  return PBICG_OK;
}

// Buffers of the peer-memory transport for one rank (zeroed flags and epoch).
double* ghost_vec(pbicg_ctx* h, int q) {  // 0 w0, 1 w1, 2 z0, 3 z1
  return q == 0 ? h->V.w0 : q == 1 ? h->V.w1 : q == 2 ? h->V.z0 : h->V.z1;
}

pbicg_status p2p_alloc(pbicg_ctx* h) {
  if (h->p2p_buf) return PBICG_OK;
  void *b = nullptr, *f = nullptr, *e = nullptr;
  ST(dalloc(h, &b, (size_t)2 * h->nranks * RED_K * sizeof(Dd)));
  ST(dalloc(h, &f, (size_t)h->nranks * sizeof(unsigned long long)));
  ST(dalloc(h, &e, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(b, 0, (size_t)2 * h->nranks * RED_K * sizeof(Dd), h->stream));
  CU(cudaMemsetAsync(f, 0, (size_t)h->nranks * sizeof(unsigned long long), h->stream));
  CU(cudaMemsetAsync(e, 0, sizeof(unsigned long long), h->stream));
  CU(cudaStreamSynchronize(h->stream));
  h->p2p_buf = (Dd*)b;
  h->p2p_flags = (unsigned long long*)f;
  h->p2p_ep = (unsigned long long*)e;
  return PBICG_OK;
}

// Peer tables: loopback members share one address space; NCCL ranks exchange
// CUDA IPC handles of their buffers with an all-gather (collective, once).
pbicg_status p2p_setup(const Members& G) {
  pbicg_ctx* h = G[0];
  if (h->nranks > P2P_MAXR)
    return fail(h, PBICG_EINVAL, "transport 1 (peer memory) supports up to 8 ranks");
  if (h->comm == COMM_LOOP) {
    for (pbicg_ctx* m : G) ST(p2p_alloc(m));
    for (size_t r = 0; r < G.size(); ++r) {
      pbicg_ctx* m = G[r];
      m->p2p_recv_tab.clear();
      m->p2p_flag_tab.clear();
      for (pbicg_ctx* q : G) {
        m->p2p_recv_tab.push_back(q->p2p_buf);
        m->p2p_flag_tab.push_back(q->p2p_flags);
      }
      for (int q = 0; q < 4; ++q) {
        m->peer_ghost[q][0] = r > 0 ? ghost_vec(G[r - 1], q) + G[r - 1]->n_local : nullptr;
        m->peer_ghost[q][1] = r + 1 < G.size() ? ghost_vec(G[r + 1], q) - G[r + 1]->halo_n
                                               : nullptr;
      }
    }
    return PBICG_OK;
  }
  if (h->comm != COMM_NCCL) return fail(h, PBICG_ESTATE, "transport 1 needs several ranks");
  if (!h->p2p_recv_tab.empty()) return PBICG_OK;
  ST(p2p_alloc(h));
  const int P = h->nranks;
  // per rank: the reduction buffer and flags, the allocations of w0, w1, z0, z1 (ghost
  // planes written by the neighbours' sweeps), and the geometry to address them
  struct Blob {
    cudaIpcMemHandle_t buf, flags, vec[4];
    int64_t n_local, halo_n, H;
  } mine{};
  CU(cudaIpcGetMemHandle(&mine.buf, h->p2p_buf));
  CU(cudaIpcGetMemHandle(&mine.flags, h->p2p_flags));
  for (int q = 0; q < 4; ++q) CU(cudaIpcGetMemHandle(&mine.vec[q], ghost_vec(h, q) - h->H));
  mine.n_local = h->n_local;
  mine.halo_n = h->halo_n;
  mine.H = h->H;
  const size_t hb = sizeof(Blob);
  void *dsend = nullptr, *drecv = nullptr;
  ST(dalloc(h, &dsend, hb));
  ST(dalloc(h, &drecv, hb * P));
  ST(upload(h, dsend, &mine, hb));
  NC(nccl_api().AllGather(dsend, drecv, hb, ncclChar, h->nccl_halo, h->stream));
  std::vector<Blob> all((size_t)P);
  CU(cudaStreamSynchronize(h->stream));
  CU(cudaMemcpy(all.data(), drecv, hb * P, cudaMemcpyDeviceToHost));
  for (int q = 0; q < P; ++q) {
    if (q == h->rank) {
      h->p2p_recv_tab.push_back(h->p2p_buf);
      h->p2p_flag_tab.push_back(h->p2p_flags);
      continue;
    }
    void *pb = nullptr, *pf = nullptr;
    CU(cudaIpcOpenMemHandle(&pb, all[q].buf, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_opened.push_back(pb);
    CU(cudaIpcOpenMemHandle(&pf, all[q].flags, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_opened.push_back(pf);
    h->p2p_recv_tab.push_back((Dd*)pb);
    h->p2p_flag_tab.push_back((unsigned long long*)pf);
    if (h->kind == KIND_STENCIL && (q == h->rank - 1 || q == h->rank + 1)) {
      const int side = q == h->rank - 1 ? 0 : 1;
      for (int v = 0; v < 4; ++v) {
        void* pv = nullptr;
        CU(cudaIpcOpenMemHandle(&pv, all[q].vec[v], cudaIpcMemLazyEnablePeerAccess));
        h->ipc_opened.push_back(pv);
        double* row0 = (double*)pv + all[q].H;  // the peer's local row 0
        h->peer_ghost[v][side] = side == 0 ? row0 + all[q].n_local : row0 - all[q].halo_n;
      }
    }
  }
  return PBICG_OK;
}

// point the tile sweeps' ghost stores at the neighbours (transport 1) or nowhere
void set_peer_halo(pbicg_ctx* h, bool on) {
  h->tg.peer = on && h->kind == KIND_STENCIL;
  for (int b = 0; b < 2; ++b)
    for (int sd = 0; sd < 2; ++sd) {
      h->V.hw[b][sd] = on ? h->peer_ghost[b][sd] : nullptr;      // w0, w1
      h->V.hz[b][sd] = on ? h->peer_ghost[2 + b][sd] : nullptr;  // z0, z1
    }
}


// NCCL communicators: the halo communicator with NCCL's defaults, the reduction
// communicator (payload 32-256 B per rank) limited to NCCL_RED_MAX_CTAS CTAs so the
// all-reduce on the side stream takes as few SMs as possible from the concurrent
// sweep / SpMV; the side stream has the device's highest priority.
// A pbicg_dist of ONE rank with an id is a real one-rank NCCL job: the same
// rank-row exchange and finalize kernels run (tests exercise the NCCL calls, graph
// capture of NCCL nodes and the peer-memory setup on one GPU).
#define NCCL_RED_MAX_CTAS 2
pbicg_status nccl_setup(pbicg_ctx* h, const pbicg_dist* d) {
  auto& api = nccl_api();
  if (!api.ok) return fail(h, PBICG_ESTATE, api.err);
  if (!d->nccl_id_halo) return fail(h, PBICG_EINVAL, "nccl_id_halo is NULL");
  ncclUniqueId id;
  memcpy(&id, d->nccl_id_halo, sizeof(id));
  NC(api.CommInitRank(&h->nccl_halo, d->nranks, id, d->rank));
  if (d->nccl_id_red) {
    memcpy(&id, d->nccl_id_red, sizeof(id));
    if (api.CommInitRankConfig) {
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.minCTAs = 1;
      cfg.maxCTAs = NCCL_RED_MAX_CTAS;
      NC(api.CommInitRankConfig(&h->nccl_red, d->nranks, id, d->rank, &cfg));
    } else {
      NC(api.CommInitRank(&h->nccl_red, d->nranks, id, d->rank));
    }
  } else {
    h->nccl_red = h->nccl_halo;
    h->overlap = 0;  // one communicator: its operations must stay on one stream
  }
  h->comm = COMM_NCCL;
  h->dist = true;
  return PBICG_OK;
}

// ------------------------- stencil construction ------------------------------
pbicg_status validate_stencil(const pbicg_stencil* op, int nranks) {
  if (!op) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  if (op->dim != 2 && op->dim != 3) return fail(nullptr, PBICG_EINVAL, "dim must be 2 or 3");
  const int64_t nz = op->dim == 3 ? op->nz : 1;
  if (op->nx < 1 || op->ny < 1 || nz < 1)
    return fail(nullptr, PBICG_EINVAL, "grid sizes must be >= 1");
  if (op->nx > (1LL << 24) || op->ny > (1LL << 24) || nz > (1LL << 24))
    return fail(nullptr, PBICG_EINVAL, "grid extent too large");
  for (int i = 0; i < 7; ++i)
    if (!std::isfinite(op->coef[i])) return fail(nullptr, PBICG_EINVAL, "non-finite coefficient");
  if (op->coef[0] == 0.0)
    return fail(nullptr, PBICG_EINVAL, "centre coefficient must be nonzero (Jacobi)");
  const int64_t outer = op->dim == 3 ? nz : op->ny;
  if (nranks < 1 || nranks > outer)
    return fail(nullptr, PBICG_EINVAL, "need 1 <= nranks <= number of slabs (nz in 3D, ny in 2D)");
  return PBICG_OK;
}

// slab partition: rank r owns outer planes [o0, o0 + nol)
void slab(int64_t outer, int nranks, int rank, int64_t* o0, int64_t* nol) {
  const int64_t base = outer / nranks, rem = outer % nranks;
  *nol = base + (rank < rem ? 1 : 0);
  *o0 = rank * base + (rank < rem ? rank : rem);
}

// Constants of the automated-replacement bound for a stencil (reading A29):
// ||A|| <= sqrt(||A||_1 ||A||_inf) with the row sums in ascending column order
// (legs -z,-y,-x,c,+x,+y,+z) and the column sums in ascending row order (the
// rows j-pxy, j-nx, j-1, j, j+1, j+nx, j+pxy contribute c[6], c[4], c[2], c[0],
// c[1], c[3], c[5]), maximised over the leg patterns that occur (first, second
// and last point of every dimension); mu = max legs per row.  Bitwise the same
// doubles as oracle.c's orc_anorm_bound on the written-out matrix.
void stencil_bound_consts(pbicg_ctx* h, const pbicg_stencil* op) {
  const int dim = op->dim;
  const int64_t n3[3] = {op->nx, op->ny, dim == 3 ? op->nz : 1};
  const double* c = op->coef;
  const int cm[3] = {1, 3, 5}, cp[3] = {2, 4, 6};  // -d / +d coefficient index
  double rmax = 0.0, cmax = 0.0;
  int64_t mu = 0;
  int64_t pos[3][3];
  int npos[3];
  for (int d = 0; d < 3; ++d) {
    npos[d] = 0;
    const int64_t cand[3] = {0, 1, n3[d] - 1};
    for (int q = 0; q < 3; ++q) {
      if (cand[q] < 0 || cand[q] >= n3[d]) continue;
      bool dup = false;
      for (int u = 0; u < npos[d]; ++u) dup |= pos[d][u] == cand[q];
      if (!dup) pos[d][npos[d]++] = cand[q];
    }
  }
  for (int a = 0; a < npos[0]; ++a)
    for (int b = 0; b < npos[1]; ++b)
      for (int e = 0; e < npos[2]; ++e) {
        const int64_t p[3] = {pos[0][a], pos[1][b], pos[2][e]};
        bool lo[3], hi[3];
        for (int d = 0; d < 3; ++d) {
          lo[d] = d < dim && p[d] > 0;
          hi[d] = d < dim && p[d] < n3[d] - 1;
        }
        // row: -z, -y, -x, c, +x, +y, +z
        double rs = 0.0;
        int64_t cnt = 1;
        for (int d = 2; d >= 0; --d)
          if (lo[d]) { rs = rs + std::fabs(c[cm[d]]); cnt++; }
        rs = rs + std::fabs(c[0]);
        for (int d = 0; d < 3; ++d)
          if (hi[d]) { rs = rs + std::fabs(c[cp[d]]); cnt++; }
        // column j: rows j-pxy (+z leg), j-nx (+y), j-1 (+x), j, j+1 (-x), j+nx (-y), j+pxy (-z)
        double cs = 0.0;
        for (int d = 2; d >= 0; --d)
          if (lo[d]) cs = cs + std::fabs(c[cp[d]]);
        cs = cs + std::fabs(c[0]);
        for (int d = 0; d < 3; ++d)
          if (hi[d]) cs = cs + std::fabs(c[cm[d]]);
        if (rs > rmax) rmax = rs;
        if (cs > cmax) cmax = cs;
        if (cnt > mu) mu = cnt;
      }
  const double n = (double)(n3[0] * n3[1] * n3[2]);
  h->ar_nA = std::sqrt(cmax * rmax);
  h->ar_muN = (double)mu * std::sqrt(n);
  h->ar_mutN = 1.0 * std::sqrt(n) * std::fabs(1.0 / c[0]);
  const int bj = h->tg.bj;
  if (bj > 1) {  // ||M^-1|| <= sqrt(||B^-1||_1 ||B^-1||_inf) of the common block (A29, A33)
    double rm = 0.0, cm = 0.0;
    for (int a = 0; a < bj; ++a) {
      double rs = 0.0;
      for (int q = 0; q < bj; ++q) rs = rs + std::fabs(h->tg.bi[a * bj + q]);
      if (rs > rm) rm = rs;
    }
    for (int q = 0; q < bj; ++q) {
      double cs = 0.0;
      for (int a = 0; a < bj; ++a) cs = cs + std::fabs(h->tg.bi[a * bj + q]);
      if (cs > cm) cm = cs;
    }
    h->ar_mutN = (double)bj * std::sqrt(n) * std::sqrt(cm * rm);
  }
  h->ar_ok = true;
}

// the common bj x bj block of a constant-coefficient stencil along x (row i: coef[1]
// at column i-1, coef[0] at i, coef[2] at i+1), inverted by the same Gauss-Jordan as
// block_inverse / oracle.c (reading A33)
pbicg_status stencil_block_inverse(const pbicg_stencil* op, int bj, double* bi) {
  std::vector<double> a((size_t)bj * bj, 0.0), e((size_t)bj * bj);
  for (int r = 0; r < bj; ++r) {
    if (r > 0) a[(size_t)r * bj + r - 1] = op->coef[1];
    a[(size_t)r * bj + r] = op->coef[0];
    if (r + 1 < bj) a[(size_t)r * bj + r + 1] = op->coef[2];
  }
  for (int r = 0; r < bj; ++r)
    for (int c = 0; c < bj; ++c) e[(size_t)r * bj + c] = (r == c) ? 1.0 : 0.0;
  for (int p = 0; p < bj; ++p) {
    const double piv = a[(size_t)p * bj + p];
    if (piv == 0.0 || !std::isfinite(piv))
      return fail(nullptr, PBICG_EINVAL, "block Jacobi: zero pivot in the stencil block");
    const double f = 1.0 / piv;
    for (int c = 0; c < bj; ++c) {
      a[(size_t)p * bj + c] = a[(size_t)p * bj + c] * f;
      e[(size_t)p * bj + c] = e[(size_t)p * bj + c] * f;
    }
    for (int r = 0; r < bj; ++r) {
      if (r == p) continue;
      const double g = a[(size_t)r * bj + p];
      for (int c = 0; c < bj; ++c) {
        a[(size_t)r * bj + c] = a[(size_t)r * bj + c] - g * a[(size_t)p * bj + c];
        e[(size_t)r * bj + c] = e[(size_t)r * bj + c] - g * e[(size_t)p * bj + c];
      }
    }
  }
  for (size_t q = 0; q < e.size(); ++q) bi[q] = e[q];
  return PBICG_OK;
}

pbicg_status build_stencil(pbicg_ctx* h, const pbicg_stencil* op, int bj) {
  h->kind = KIND_STENCIL;
  h->tg.bj = 1;
  if (bj > 1) {
    if (op->nx % bj != 0)
      return fail(h, PBICG_EINVAL, "block Jacobi on a stencil needs nx % b == 0");
    if (op->nx > 1024)
      return fail(h, PBICG_EINVAL, "block Jacobi on a stencil needs nx <= 1024 (tile kernels)");
    ST(stencil_block_inverse(op, bj, h->tg.bi));
    h->tg.bj = bj;
  }
  stencil_bound_consts(h, op);
  h->dim = op->dim;
  const int64_t nz = op->dim == 3 ? op->nz : 1;
  Geo& g = h->geo;
  g.nx = op->nx;
  g.ny = op->ny;
  const int64_t outer = op->dim == 3 ? nz : op->ny;
  g.nog = outer;
  slab(outer, h->nranks, h->rank, &g.o0, &g.nol);
  g.pxy = op->dim == 3 ? op->nx * op->ny : op->nx;
  g.nlines = op->dim == 3 ? op->ny * g.nol : g.nol;
  for (int i = 0; i < 7; ++i) g.c[i] = op->coef[i];
  if (op->dim == 2) {
    g.c[5] = 0.0;
    g.c[6] = 0.0;
  }
  g.dinv = 1.0 / op->coef[0];  // A3
  h->n_global = op->nx * op->ny * nz;
  h->n_local = g.pxy * g.nol;
  h->row_begin = g.o0 * g.pxy;
  // ghost plane + staging slack of the tile kernels (segmented tiles stage line y-1,
  // column x-SEG_HX of plane -1: pxy + nx + 8 before, pxy + nx + 6 after)
  h->H = g.pxy + g.nx + 2 * SEG_HX;
  h->halo_n = g.pxy;
  h->block = 256;
  if (g.nx < 256) h->block = (int)(((g.nx + 31) / 32) * 32);
  if (h->block < 64) h->block = 64;
  const int64_t L = g.nlines;
  if (op->dim == 3) {
    h->grid[K_INIT] = occ_grid(h, k_init1<3>, L);
    h->grid[K_SWEEPA] = occ_grid(h, k_sweepA<3>, L);
    h->grid[K_SWEEPC] = occ_grid(h, k_sweepC<3>, L);
    h->grid[K_RR1] = occ_grid(h, k_rr1<3>, L);
    h->grid[K_RR2] = occ_grid(h, k_rr2<3>, L);
    h->grid[K_GAP] = occ_grid(h, k_gap<3>, L);
    h->grid[K_APPLY] = occ_grid(h, k_apply<3>, L);
    { const int b0 = h->block; h->block = 256;
      h->grid_a2 = occ_grid(h, k_sweepA2<3>, (h->n_local + 255) / 256);
      h->grid_c2 = occ_grid(h, k_sweepC2<3>, (h->n_local + 255) / 256); h->block = b0; }
  } else {
    h->grid[K_INIT] = occ_grid(h, k_init1<2>, L);
    h->grid[K_SWEEPA] = occ_grid(h, k_sweepA<2>, L);
    h->grid[K_SWEEPC] = occ_grid(h, k_sweepC<2>, L);
    h->grid[K_RR1] = occ_grid(h, k_rr1<2>, L);
    h->grid[K_RR2] = occ_grid(h, k_rr2<2>, L);
    h->grid[K_GAP] = occ_grid(h, k_gap<2>, L);
    h->grid[K_APPLY] = occ_grid(h, k_apply<2>, L);
    { const int b0 = h->block; h->block = 256;
      h->grid_a2 = occ_grid(h, k_sweepA2<2>, (h->n_local + 255) / 256);
      h->grid_c2 = occ_grid(h, k_sweepC2<2>, (h->n_local + 255) / 256); h->block = b0; }
  }
  {  // split schedule (option schedule 2): point-wise sweeps on the TMA chunk ring
    const auto SM = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaFuncSetAttribute(c_sweep_tma<0, false, false, true>, SM, (int)kCstSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(c_sweep_tma<1, false, false, true>, SM, (int)kCstSmem);
    h->csr.n = h->n_local;  // the kernel's row count (no matrix on a stencil handle)
    h->csr.bj = 1;
    const int64_t nch = (h->n_local + CST_R - 1) / CST_R;
    h->cst_grid = (int)(nch < h->num_sm ? nch : h->num_sm);
    h->cst_ok = e == cudaSuccess && h->H % 2 == 0;  // 16-byte aligned row pairs
    cudaGetLastError();
  }
  setup_tile(h);
  constexpr int64_t kSplitRows = 3000000;  // see split_sched
  if (h->comm == COMM_NCCL && h->nranks > 1 && bj <= 1 && h->tile_ok && h->n_local < kSplitRows &&
      !getenv("PBICG_NO_AUTO_SPLIT"))
    h->auto_split = true;
  if (bj > 1 && (!h->tile_ok || h->tile_seg))
    return fail(h, PBICG_EINVAL,
                "block Jacobi on a stencil needs full-line TMA tiles (2D: nx <= 1024, "
                "3D: nx <= ~850)");
  ST(alloc_common(h));
  if (h->auto_split) {  // stored t, v of the split schedule
    ST(gvec(h, &h->V.tv));
    ST(gvec(h, &h->V.vv));
  }
  return PBICG_OK;
}

// ---------------------------- CSR construction --------------------------------
pbicg_status validate_csr(const pbicg_csr* op, int nranks, std::vector<double>* dinv,
                          int64_t* width, bool* uniform, int64_t halo = PBICG_CSR_HALO) {
  if (!op || !op->row_ptr || (op->n_local > 0 && (!op->col || !op->val)))
    return fail(nullptr, PBICG_EINVAL, "NULL argument");
  const int64_t n = op->n_local;
  if (op->n_global < 1 || n < 1 || op->row_begin < 0 || op->row_begin + n > op->n_global)
    return fail(nullptr, PBICG_EINVAL, "bad row range");
  if (op->n_global > INT32_MAX) return fail(nullptr, PBICG_EINVAL, "n_global must fit int32");
  const int64_t H = nranks > 1 ? halo : 0;
  if (nranks == 1 && (op->row_begin != 0 || n != op->n_global))
    return fail(nullptr, PBICG_EINVAL, "single rank: the rank must own all rows");
  if (nranks > 1 && n < H)
    return fail(nullptr, PBICG_EINVAL, "multi-rank CSR: every rank needs >= halo (PBICG_CSR_HALO) rows");
  const int64_t lo = op->row_begin - H, hi = op->row_begin + n + H;
  const int64_t* rp = op->row_ptr;
  *width = 0;
  *uniform = true;
  dinv->assign(n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t len = rp[i + 1] - rp[i];
    if (len < 1) return fail(nullptr, PBICG_EINVAL, "row without entries (needs a diagonal)");
    if (i > 0 && len != *width) *uniform = false;
    if (len > *width) *width = len;
    bool diag = false;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = op->col[p];
      if (c < 0 || c >= op->n_global) return fail(nullptr, PBICG_EINVAL, "column out of range");
      if (c < lo || c >= hi)
        return fail(nullptr, PBICG_EINVAL, "column outside the nearest-neighbour halo band");
      if (p > rp[i] && c <= op->col[p - 1])
        return fail(nullptr, PBICG_EINVAL, "columns must be strictly ascending within a row");
      if (!std::isfinite(op->val[p])) return fail(nullptr, PBICG_EINVAL, "non-finite value");
      if (c == op->row_begin + i) {
        if (op->val[p] == 0.0)
          return fail(nullptr, PBICG_EINVAL, "zero diagonal (Jacobi undefined)");
        (*dinv)[i] = 1.0 / op->val[p];  // A3
        diag = true;
      }
    }
    if (!diag) return fail(nullptr, PBICG_EINVAL, "missing diagonal entry");
  }
  if (*width > 4096) return fail(nullptr, PBICG_EINVAL, "row too long for the ELL path (> 4096)");
  return PBICG_OK;
}

// Block Jacobi (reading A33): the bj x bj diagonal blocks of this rank's rows
// (rows [k bj, (k+1) bj), aligned globally), each inverted by plain Gauss-Jordan
// elimination without pivoting -- the same operations, in the same order, as
// oracle.c orc_gauss_jordan -- stored row-major as binv[i * bj + c].
pbicg_status block_inverse(const pbicg_csr* op, int bj, std::vector<double>* binv) {
  const int64_t n = op->n_local;
  binv->assign((size_t)n * bj, 0.0);
  std::vector<double> a((size_t)bj * bj), e((size_t)bj * bj);
  for (int64_t k0 = 0; k0 < n; k0 += bj) {
    std::fill(a.begin(), a.end(), 0.0);
    for (int r = 0; r < bj; ++r)
      for (int64_t p = op->row_ptr[k0 + r]; p < op->row_ptr[k0 + r + 1]; ++p) {
        const int64_t c = op->col[p] - op->row_begin - k0;
        if (c >= 0 && c < bj) a[(size_t)r * bj + c] = op->val[p];
      }
    for (int r = 0; r < bj; ++r)
      for (int c = 0; c < bj; ++c) e[(size_t)r * bj + c] = (r == c) ? 1.0 : 0.0;
    for (int p = 0; p < bj; ++p) {
      const double piv = a[(size_t)p * bj + p];
      if (piv == 0.0 || !std::isfinite(piv))
        return fail(nullptr, PBICG_EINVAL, "block Jacobi: zero pivot in a diagonal block");
      const double f = 1.0 / piv;
      for (int c = 0; c < bj; ++c) {
        a[(size_t)p * bj + c] = a[(size_t)p * bj + c] * f;
        e[(size_t)p * bj + c] = e[(size_t)p * bj + c] * f;
      }
      for (int r = 0; r < bj; ++r) {
        if (r == p) continue;
        const double g = a[(size_t)r * bj + p];
        for (int c = 0; c < bj; ++c) {
          a[(size_t)r * bj + c] = a[(size_t)r * bj + c] - g * a[(size_t)p * bj + c];
          e[(size_t)r * bj + c] = e[(size_t)r * bj + c] - g * e[(size_t)p * bj + c];
        }
      }
    }
    for (int r = 0; r < bj; ++r)
      for (int c = 0; c < bj; ++c) (*binv)[(size_t)(k0 + r) * bj + c] = e[(size_t)r * bj + c];
  }
  return PBICG_OK;
}

// preconditioner block size from the ABI value: 1 Jacobi, b for PBICG_PREC_BJ(b)
int prec_block(int prec) {
  if (prec == PBICG_PREC_JACOBI) return 1;
  const int b = prec & 0xff;
  if ((prec & ~0xff) == PBICG_PREC_BLOCK_JACOBI && (b == 2 || b == 4 || b == 8 || b == 16 || b == 32))
    return b;
  return 0;
}

// Automated-replacement constants of a CSR operator given ALL its row blocks in
// order (reading A29): ||A|| <= sqrt(||A||_1 ||A||_inf), row sums in stored
// (ascending column) order, column sums in ascending row order -- the same
// doubles as oracle.c orc_anorm_bound; mu = max row length; ||M^-1|| = max |1/a_jj|.
// max over one rank's diagonal blocks of sqrt(||B^-1||_1 ||B^-1||_inf), row / column
// sums in ascending order (oracle prec_norm_bound)
double block_inv_norm_max(const pbicg_csr* op, int bj) {
  std::vector<double> inv;
  double mi = 0.0;
  if (block_inverse(op, bj, &inv) != PBICG_OK) return 0.0;
  for (int64_t k0 = 0; k0 < op->n_local; k0 += bj) {
    double rm = 0.0, cm = 0.0;
    for (int a = 0; a < bj; ++a) {
      double rs = 0.0;
      for (int c = 0; c < bj; ++c) rs = rs + std::fabs(inv[(size_t)(k0 + a) * bj + c]);
      if (rs > rm) rm = rs;
    }
    for (int c = 0; c < bj; ++c) {
      double cs = 0.0;
      for (int a = 0; a < bj; ++a) cs = cs + std::fabs(inv[(size_t)(k0 + a) * bj + c]);
      if (cs > cm) cm = cs;
    }
    const double nbk = std::sqrt(cm * rm);
    if (nbk > mi) mi = nbk;
  }
  return mi;
}

void csr_bound_consts(const pbicg_csr* ops, int nops, int bj, double* nA, double* muN,
                      double* mutN) {
  const int64_t N = ops[0].n_global;
  std::vector<double> col((size_t)N, 0.0);
  double rmax = 0.0, cmax = 0.0, mi = 0.0;
  int64_t mu = 0;
  for (int r = 0; r < nops; ++r) {
    const pbicg_csr& op = ops[r];
    for (int64_t i = 0; i < op.n_local; ++i) {
      double rs = 0.0;
      const int64_t p0 = op.row_ptr[i], p1 = op.row_ptr[i + 1];
      if (p1 - p0 > mu) mu = p1 - p0;
      for (int64_t p = p0; p < p1; ++p) {
        rs = rs + std::fabs(op.val[p]);
        col[(size_t)op.col[p]] = col[(size_t)op.col[p]] + std::fabs(op.val[p]);
        if (op.col[p] == op.row_begin + i && std::fabs(1.0 / op.val[p]) > mi)
          mi = std::fabs(1.0 / op.val[p]);
      }
      if (rs > rmax) rmax = rs;
    }
  }
  for (double c : col) cmax = c > cmax ? c : cmax;
  if (bj > 1) {  // ||M^-1|| <= max over blocks sqrt(||B^-1||_1 ||B^-1||_inf) (oracle prec_norm_bound)
    mi = 0.0;
    for (int r = 0; r < nops; ++r) {
      const double m = block_inv_norm_max(&ops[r], bj);
      if (m > mi) mi = m;
    }
  }
  *nA = std::sqrt(cmax * rmax);
  *muN = (double)mu * std::sqrt((double)N);
  *mutN = (double)bj * std::sqrt((double)N) * mi;
}

pbicg_status ilu_setup(pbicg_ctx* h, const pbicg_csr* op, const pbicg_stencil* st);

// The same constants computed rank by rank (multi-process CSR, reading A29): the
// column sums are accumulated in ascending row order ACROSS ranks by passing a
// window of partial column sums down the ranks -- rank r receives the sums of
// ranks < r for columns [rb - H, rb + H) (the only columns ranks < r reach that r
// reaches too; every rank holds >= H rows), adds its own rows, and hands
// [re - H, re + H) to rank r + 1.  Column j's sum is final at the rank whose range
// [rb - H, re - H) (the last rank: up to N) holds j, so the maximum over those
// ranges, combined with the row-sum / mu / ||M^-1|| maxima by an exact max
// all-reduce, is bitwise csr_bound_consts over all rows.  part = {max column sum,
// max row sum, mu, ||M^-1|| bound} of this rank.
void csr_bound_chain_step(const pbicg_csr* op, int bj, int64_t H, bool last,
                          const double* win_in, double* win_out, double part[4]) {
  const int64_t n = op->n_local, rb = op->row_begin;
  std::vector<double> acc((size_t)(n + 2 * H), 0.0);  // columns [rb - H, rb + n + H)
  if (win_in)
    for (int64_t q = 0; q < 2 * H; ++q) acc[(size_t)q] = win_in[q];
  double rmax = 0.0, mi = 0.0;
  int64_t mu = 0;
  for (int64_t i = 0; i < n; ++i) {
    double rs = 0.0;
    const int64_t p0 = op->row_ptr[i], p1 = op->row_ptr[i + 1];
    if (p1 - p0 > mu) mu = p1 - p0;
    for (int64_t p = p0; p < p1; ++p) {
      rs = rs + std::fabs(op->val[p]);
      double& c = acc[(size_t)(op->col[p] - (rb - H))];
      c = c + std::fabs(op->val[p]);
      if (op->col[p] == rb + i && std::fabs(1.0 / op->val[p]) > mi) mi = std::fabs(1.0 / op->val[p]);
    }
    if (rs > rmax) rmax = rs;
  }
  if (bj > 1) mi = block_inv_norm_max(op, bj);  // ||M^-1|| over this rank's blocks
  const int64_t fin = last ? n + H : n;  // final column range [rb - H, rb - H + fin)
  double cmax = 0.0;
  for (int64_t q = 0; q < fin; ++q) cmax = acc[(size_t)q] > cmax ? acc[(size_t)q] : cmax;
  if (win_out)
    for (int64_t q = 0; q < 2 * H; ++q) win_out[q] = acc[(size_t)(n + q)];
  part[0] = cmax;
  part[1] = rmax;
  part[2] = (double)mu;
  part[3] = mi;
}

void bound_consts_from_parts(const double* parts, int P, int64_t N, int bj, double* nA,
                             double* muN, double* mutN) {
  double c = 0, r = 0, mu = 0, mi = 0;
  for (int q = 0; q < P; ++q) {
    c = parts[4 * q] > c ? parts[4 * q] : c;
    r = parts[4 * q + 1] > r ? parts[4 * q + 1] : r;
    mu = parts[4 * q + 2] > mu ? parts[4 * q + 2] : mu;
    mi = parts[4 * q + 3] > mi ? parts[4 * q + 3] : mi;
  }
  *nA = std::sqrt(c * r);
  *muN = mu * std::sqrt((double)N);
  *mutN = (double)bj * std::sqrt((double)N) * mi;
}

pbicg_status build_csr(pbicg_ctx* h, const pbicg_csr* op, const std::vector<double>& dinv,
                       int64_t width, bool uniform, int bj, int ilu = 0,
                       const pbicg_stencil* st = nullptr, int64_t halo = PBICG_CSR_HALO) {
  h->kind = KIND_CSR;
  h->ilu = ilu;
  if (bj > 1) {
    if (op->n_local % bj != 0 || op->row_begin % bj != 0)
      return fail(h, PBICG_EINVAL, "block Jacobi: rank rows must be whole aligned blocks");
    std::vector<double> inv;
    ST(block_inverse(op, bj, &inv));
    void* pb = nullptr;
    ST(dalloc(h, &pb, inv.size() * sizeof(double)));
    ST(upload(h, pb, inv.data(), inv.size() * sizeof(double)));
    h->csr.binv = (const double*)pb;
  }
  h->csr.bj = bj;
  if (h->nranks == 1) {  // multi-rank: the loopback group sets them (NCCL ranks: not available)
    csr_bound_consts(op, 1, bj, &h->ar_nA, &h->ar_muN, &h->ar_mutN);
    h->ar_ok = true;
  }
  const int64_t n = op->n_local;
  const int64_t* rp = op->row_ptr;
  h->n_global = op->n_global;
  h->n_local = n;
  h->row_begin = op->row_begin;
  h->H = h->nranks > 1 ? halo : 0;
  h->halo_n = h->H;
  h->block = 256;
  // column-major ELL in stored row order; padding slots are never read (len[])
  std::vector<int32_t> ecol((size_t)width * n);
  std::vector<double> eval((size_t)width * n, 0.0);
  std::vector<int32_t> elen(uniform ? 0 : n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t len = rp[i + 1] - rp[i];
    if (!uniform) elen[i] = (int32_t)len;
    for (int64_t q = 0; q < width; ++q) {
      const bool real = q < len;
      ecol[(size_t)q * n + i] = real ? (int32_t)(op->col[rp[i] + q] - op->row_begin) : (int32_t)i;
      eval[(size_t)q * n + i] = real ? op->val[rp[i] + q] : 0.0;
    }
  }
  void *pc = nullptr, *pv = nullptr, *pl = nullptr;
  ST(dalloc(h, &pc, ecol.size() * sizeof(int32_t)));
  ST(dalloc(h, &pv, eval.size() * sizeof(double)));
  if (!uniform) ST(dalloc(h, &pl, (size_t)n * sizeof(int32_t)));
  ST(upload(h, pc, ecol.data(), ecol.size() * sizeof(int32_t)));
  ST(upload(h, pv, eval.data(), eval.size() * sizeof(double)));
  if (!uniform)
    ST(upload(h, pl, elen.data(), (size_t)n * sizeof(int32_t)));
  ST(gvec(h, &h->dinv_g));
  ST(upload(h, h->dinv_g, dinv.data(), (size_t)n * sizeof(double)));
  h->csr.n = n;
  h->csr.width = (int32_t)width;
  h->csr.col = (const int32_t*)pc;
  h->csr.val = (const double*)pv;
  h->csr.len = uniform ? nullptr : (const int32_t*)pl;
  h->csr.dinv = h->dinv_g;
  const int64_t blocks = (n + h->block - 1) / h->block;
  // (the NRM variants reuse these grids: grid-stride loops, last-CTA reductions)
  h->grid[K_INIT] = occ_grid(h, c_init1<false, PK_JAC>, blocks);
  h->grid[K_SWEEPA] = occ_grid(h, c_sweepA<false, PK_JAC>, blocks);
  h->grid[K_SWEEPC] = occ_grid(h, c_sweepC<false, PK_JAC>, blocks);
  h->grid[K_SPMVB] = occ_grid(h, c_spmvB, blocks);
  h->grid[K_SPMVD] = occ_grid(h, c_spmvD, blocks);
  h->grid[K_RR1] = occ_grid(h, c_rr1<false, PK_JAC>, blocks);
  h->grid[K_RR2] = occ_grid(h, c_rr2<false, PK_JAC>, blocks);
  h->grid[K_GAP] = occ_grid(h, c_gap, blocks);
  h->grid[K_APPLY] = occ_grid(h, c_apply, blocks);
  ST(gvec(h, &h->V.nv));
  ST(gvec(h, &h->V.mv));
  // window SpMV: half bandwidth of this rank's rows, ring of WRS doubles
  int64_t bw = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      const int64_t d = op->col[q] - (op->row_begin + i);
      bw = d < 0 ? (-d > bw ? -d : bw) : (d > bw ? d : bw);
    }
  // the window's first element R0 - bw must be 16-byte aligned for the bulk copies:
  // round the half bandwidth up to even (rows of an odd band just stage one more column)
  bw = (bw + 1) & ~(int64_t)1;
  // ... and so must the ghosted operand's local part: with an odd ghost width H (a rank's
  // odd stencil plane) every chunk start R0 - bw + H and the first ring position off - H
  // are odd -- such handles keep the gather SpMV (found by the randomised ILU shapes:
  // 35 x 47 x 3 on three loopback ranks faulted with "misaligned address")
  if (3LL * WTB + 2 * bw <= WRS && h->H % 2 == 0) {
    // the window SpMV's operands as sliced ELL (SELL-32) with 16-bit column offsets
    // (|col - row| <= bw < 2^15): 10 bytes per slot, immediate-offset loads
    const int64_t ns = (n + 31) / 32;
    std::vector<double> sval((size_t)ns * width * 32, 0.0);
    std::vector<int16_t> sdcol((size_t)ns * width * 32, 0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t q = 0; q < width; ++q) {
        const size_t e = ((size_t)(i / 32) * width + q) * 32 + (i % 32);
        sval[e] = eval[(size_t)q * n + i];
        sdcol[e] = (int16_t)(ecol[(size_t)q * n + i] - i);
      }
    void *psv = nullptr, *psd = nullptr;
    ST(dalloc(h, &psv, sval.size() * sizeof(double)));
    ST(dalloc(h, &psd, sdcol.size() * sizeof(int16_t)));
    ST(upload(h, psv, sval.data(), sval.size() * sizeof(double)));
    ST(upload(h, psd, sdcol.data(), sdcol.size() * sizeof(int16_t)));
    h->csr.sval = (const double*)psv;
    h->csr.sdcol = (const int16_t*)psd;
    WinGeo& w = h->wg;
    w.bw = (int32_t)bw;
    w.lo = -h->H;
    w.hi = n + h->H;
    w.off = ((h->H + WTB - 1) / WTB) * WTB;
    int64_t per = (n + h->num_sm - 1) / h->num_sm;
    per = ((per + WTB - 1) / WTB) * WTB;
    w.rows_cta = (int32_t)per;
    h->win_grid = (int)((n + per - 1) / per);
    const cudaFuncAttribute SM = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaFuncSetAttribute(c_spmv_win<SP_V>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_T>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_CLS>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_CLY>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_PCW0>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_PCN>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_GAP>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_I1>, SM, WIN_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_spmv_win<SP_I2>, SM, WIN_SMEM);
    h->win_ok = e == cudaSuccess;
    cudaGetLastError();
  }
  // TMA-staged sweeps: one CTA per SM, two-stage chunk ring.  Block Jacobi b <= 4 only:
  // measured on cfg5 (it/s, per-row kernel -> TMA ring) b = 2: 781 -> 834, b = 4: 757 ->
  // 761, b = 8: 673 -> 570 (the per-thread gathers of two b-wide inverse rows lack the
  // per-row kernel's 24 warps per SM of memory parallelism), b = 16, 32 likewise slower
  if (h->csr.bj <= 4) {
    const auto SM = cudaFuncAttributeMaxDynamicSharedMemorySize;
    const int sm = (int)kCstSmem;
    cudaError_t e = cudaFuncSetAttribute(c_sweep_tma<0, false, false>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<0, true, false>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<1, false, false>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<1, true, false>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<0, false, true>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<0, true, true>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<1, false, true>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_sweep_tma<1, true, true>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_cl_tma<0>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_cl_tma<1>, SM, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(c_cl_tma<2>, SM, sm);
    const int64_t nch = (n + CST_R - 1) / CST_R;
    h->cst_grid = (int)(nch < h->num_sm ? nch : h->num_sm);
    h->cst_ok = e == cudaSuccess && h->H % 2 == 0;  // 16-byte aligned row pairs
    cudaGetLastError();
  }
  ST(alloc_common(h));
  if (ilu) ST(ilu_setup(h, op, st));
  return PBICG_OK;
}

// ------------------------------ ILU(0) / ICC(0) ---------------------------------
// ILU(0) of this rank's diagonal block (reading A34): Saad's IKJ Gaussian elimination
// restricted to the pattern (columns of other ranks dropped), pivots as reciprocals --
// the same operations in the same order as oracle.c orc_ilu0_factor (a row's entries
// are located through a scatter map instead of a search: same arithmetic).
// lu[p] (p indexes op's entries) = l_ik below the diagonal, u_ij on / above it.
pbicg_status ilu0_host(const pbicg_csr* op, std::vector<double>* lu, std::vector<double>* uinv) {
  const int64_t n = op->n_local, rb = op->row_begin, p0 = op->row_ptr[0];
  const int64_t* rp = op->row_ptr;
  const int64_t nnz = rp[n] - p0;
  lu->assign(op->val, op->val + nnz);
  uinv->assign((size_t)n, 0.0);
  std::vector<int64_t> pos((size_t)n, -1);
  double* L = lu->data();
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = op->col[p] - rb;
      if (c >= 0 && c < n) pos[(size_t)c] = p - p0;
    }
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t k = op->col[p] - rb;
      if (k < 0) continue;
      if (k >= i) break;
      const int64_t pk = p - p0;
      L[pk] = L[pk] * (*uinv)[(size_t)k];
      for (int64_t q = rp[k]; q < rp[k + 1]; ++q) {
        const int64_t j = op->col[q] - rb;
        if (j <= k || j >= n) continue;
        const int64_t pj = pos[(size_t)j];
        if (pj >= 0) L[pj] = L[pj] - L[pk] * L[q - p0];
      }
    }
    const int64_t pd = pos[(size_t)i];
    if (pd < 0 || L[pd] == 0.0 || !std::isfinite(L[pd]))
      return fail(nullptr, PBICG_EINVAL, "ILU(0): zero or non-finite pivot in row " +
                                             std::to_string(rb + i));
    (*uinv)[(size_t)i] = 1.0 / L[pd];
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = op->col[p] - rb;
      if (c >= 0 && c < n) pos[(size_t)c] = -1;
    }
  }
  return PBICG_OK;
}

// ICC(0) needs a symmetric diagonal block (the block M is built from)
bool block_symmetric(const pbicg_csr* op) {
  const int64_t n = op->n_local, rb = op->row_begin;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = op->row_ptr[i]; p < op->row_ptr[i + 1]; ++p) {
      const int64_t c = op->col[p] - rb;
      if (c < 0 || c >= n) continue;
      const int32_t* b = op->col + op->row_ptr[c];
      const int32_t* e = op->col + op->row_ptr[c + 1];
      const int32_t* f = std::lower_bound(b, e, (int32_t)(rb + i));
      if (f == e || *f != rb + i || op->val[op->row_ptr[c] + (f - b)] != op->val[p]) return false;
    }
  return true;
}

pbicg_status ilu_setup(pbicg_ctx* h, const pbicg_csr* op, const pbicg_stencil* st) {
  std::vector<double> lu, uinv;
  ST(ilu0_host(op, &lu, &uinv));
  const int64_t n = op->n_local, rb = op->row_begin, p0 = op->row_ptr[0];
  const int64_t* rp = op->row_ptr;
  IluOp& P = h->ilu_op;
  void* pu = nullptr;
  ST(dalloc(h, &pu, (size_t)n * sizeof(double)));
  ST(upload(h, pu, uinv.data(), (size_t)n * sizeof(double)));
  P.uinv = (const double*)pu;
  void* pc = nullptr;
  ST(dalloc(h, &pc, 8 * sizeof(unsigned int)));
  CU(cudaMemsetAsync(pc, 0, 8 * sizeof(unsigned int), h->stream));
  P.ctr = (unsigned int*)pc;
  P.n = n;
  // stencil: the wavefront kernels recompute l_ik = fl(c_leg uinv_k) and u_ij = c_leg;
  // confirm the factors are exactly that (no fill interaction on a 5/7-point stencil)
  bool st_ok = st != nullptr;
  if (st_ok) {
    const double* c = st->coef;
    for (int64_t i = 0; i < n && st_ok; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int64_t k = op->col[p] - rb;
        if (k < 0 || k >= n || k == i) continue;
        const int64_t d = i - k;  // > 0: lower leg
        const int leg = d == 1 ? 1 : d == -1 ? 2 : d == st->nx ? 3 : d == -st->nx ? 4
                        : d > 0 ? 5 : 6;
        const double want = d > 0 ? c[leg] * uinv[(size_t)k] : c[leg];
        if (lu[(size_t)(p - p0)] != want) { st_ok = false; break; }
      }
  }
  // k_ilu_st addresses a tile's rows by 32-bit offsets: (ILU_BMAX + 1) planes and lines
  // must stay below 2^30 rows (else the general CSR sweeps run)
  if (st_ok && st->dim == 3 &&
      (int64_t)(ILU_BMAX + 1) * (st->nx * st->ny + st->nx) + st->nx >= ((int64_t)1 << 30))
    st_ok = false;
  h->ilu_st = st_ok;
  if (st_ok) {
    const Geo& g = h->geo;  // set by the stencil create path
    P.dim = st->dim;
    P.nx = st->nx;
    P.cxm = st->coef[1];
    P.cxp = st->coef[2];
    P.cam = st->coef[3];
    P.cap = st->coef[4];
    if (st->dim == 3) {
      P.na = st->ny;
      P.nb = g.nol;
      P.sa = st->nx;
      P.sb = st->nx * st->ny;
      P.cbm = st->coef[5];
      P.cbp = st->coef[6];
      int64_t ta = 16;
      if (const char* e = getenv("PBICG_ILU_TA")) {  // tuning experiments only
        const long v = strtol(e, nullptr, 10);
        if (v >= 1 && v <= ILU_BMAX) ta = v;  // boundary-value slots per side
      }
      P.TA = (int32_t)(st->ny < ta ? st->ny : ta);
      int64_t tb = ILU_T / P.TA;
      if (tb > ILU_BMAX) tb = ILU_BMAX;  // boundary-value slots per side
      P.TB = (int32_t)(g.nol < tb ? g.nol : tb);
    } else {
      P.na = g.nol;
      P.nb = 1;
      P.sa = st->nx;
      P.sb = 0;
      P.cbm = P.cbp = 0.0;
      P.TA = 32 * I2_W;  // k_ilu_2d: I2_W warps of 32 lines
      P.TB = 1;
    }
    P.nta = (int32_t)((P.na + P.TA - 1) / P.TA);
    P.ntb = (int32_t)((P.nb + P.TB - 1) / P.TB);
    P.ntiles = P.nta * P.ntb;
    std::vector<int32_t> order;  // diagonals of the tile grid, then A
    for (int32_t d = 0; d <= P.nta + P.ntb - 2; ++d)
      for (int32_t A = 0; A < P.nta; ++A) {
        const int32_t B = d - A;
        if (B >= 0 && B < P.ntb) order.push_back(A + P.nta * B);
      }
    void *po = nullptr, *pf = nullptr, *pb = nullptr;
    ST(dalloc(h, &po, order.size() * sizeof(int32_t)));
    ST(upload(h, po, order.data(), order.size() * sizeof(int32_t)));
    ST(dalloc(h, &pf, (size_t)P.ntiles * sizeof(unsigned long long)));
    ST(dalloc(h, &pb, (size_t)P.ntiles * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(pf, 0, (size_t)P.ntiles * sizeof(unsigned long long), h->stream));
    CU(cudaMemsetAsync(pb, 0, (size_t)P.ntiles * sizeof(unsigned long long), h->stream));
    CU(cudaStreamSynchronize(h->stream));
    P.order = (const int32_t*)po;
    P.prog_f = (unsigned long long*)pf;
    P.prog_b = (unsigned long long*)pb;
    const auto SMA = cudaFuncAttributeMaxDynamicSharedMemorySize;
    CU(cudaFuncSetAttribute(k_ilu_st<3, false>, SMA, (int)kIluSmem));
    CU(cudaFuncSetAttribute(k_ilu_st<3, true>, SMA, (int)kIluSmem));
    int occ = 0, occ_max = 0;
    if (P.dim == 3) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_max, k_ilu_st<3, false>, kIluThreads, kIluSmem);
      occ = ILU_OCC3 < occ_max ? ILU_OCC3 : occ_max;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_max, k_ilu_2d<false>, 32 * I2_W, 0);
      occ = occ_max;
    }
    if (const char* e = getenv("PBICG_ILU_OCC")) {  // tuning experiments only
      const long v = strtol(e, nullptr, 10);
      if (v >= 1 && v <= occ_max) occ = (int)v;
    }
    const int64_t cap = (int64_t)(occ < 1 ? 1 : occ) * h->num_sm;
    h->ilu_grid = (int)(P.ntiles < cap ? P.ntiles : cap);
    return PBICG_OK;
  }
  // general CSR: strictly lower / upper parts as column-major ELL, level orders
  std::vector<int32_t> nl((size_t)n, 0), nu((size_t)n, 0), lev((size_t)n, 0), levb((size_t)n, 0);
  int32_t wl = 0, wu = 0, nlev = 0, nlevb = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t l = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = op->col[p] - rb;
      if (c < 0 || c >= n || c == i) continue;
      if (c < i) { nl[(size_t)i]++; l = std::max(l, lev[(size_t)c] + 1); }
      else nu[(size_t)i]++;
    }
    lev[(size_t)i] = l;
    nlev = std::max(nlev, l + 1);
    wl = std::max(wl, nl[(size_t)i]);
    wu = std::max(wu, nu[(size_t)i]);
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    int32_t l = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = op->col[p] - rb;
      if (c > i && c < n) l = std::max(l, levb[(size_t)c] + 1);
    }
    levb[(size_t)i] = l;
    nlevb = std::max(nlevb, l + 1);
  }
  std::vector<int32_t> lcol((size_t)wl * n, -1), ucol((size_t)wu * n, -1);
  std::vector<double> lval((size_t)wl * n, 0.0), uval((size_t)wu * n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    int32_t a = 0, b = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t c = op->col[p] - rb;
      if (c < 0 || c >= n || c == i) continue;
      if (c < i) {
        lcol[(size_t)a * n + i] = (int32_t)c;
        lval[(size_t)a * n + i] = lu[(size_t)(p - p0)];
        a++;
      } else {
        ucol[(size_t)b * n + i] = (int32_t)c;
        uval[(size_t)b * n + i] = lu[(size_t)(p - p0)];
        b++;
      }
    }
  }
  // counting sort by level (forward: ascending rows within a level; backward: descending)
  std::vector<int64_t> cnt((size_t)nlev + 1, 0), cntb((size_t)nlevb + 1, 0);
  for (int64_t i = 0; i < n; ++i) { cnt[(size_t)lev[(size_t)i] + 1]++; cntb[(size_t)levb[(size_t)i] + 1]++; }
  for (size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
  for (size_t k = 1; k < cntb.size(); ++k) cntb[k] += cntb[k - 1];
  std::vector<int32_t> ford((size_t)n), bord((size_t)n);
  for (int64_t i = 0; i < n; ++i) ford[(size_t)cnt[(size_t)lev[(size_t)i]]++] = (int32_t)i;
  for (int64_t i = n - 1; i >= 0; --i) bord[(size_t)cntb[(size_t)levb[(size_t)i]]++] = (int32_t)i;
  auto up = [&](const void* src, size_t bytes, void** dst) -> pbicg_status {
    ST(dalloc(h, dst, bytes));
    if (bytes) ST(upload(h, *dst, src, bytes));
    return PBICG_OK;
  };
  void *a1, *a2, *a3, *a4, *a5, *a6, *a7;
  ST(up(lcol.data(), lcol.size() * sizeof(int32_t), &a1));
  ST(up(lval.data(), lval.size() * sizeof(double), &a2));
  ST(up(ucol.data(), ucol.size() * sizeof(int32_t), &a3));
  ST(up(uval.data(), uval.size() * sizeof(double), &a4));
  ST(up(ford.data(), ford.size() * sizeof(int32_t), &a5));
  ST(up(bord.data(), bord.size() * sizeof(int32_t), &a6));
  ST(dalloc(h, &a7, (size_t)n * sizeof(unsigned int)));
  CU(cudaMemsetAsync(a7, 0, (size_t)n * sizeof(unsigned int), h->stream));
  CU(cudaStreamSynchronize(h->stream));
  P.wl = wl;
  P.wu = wu;
  P.lcol = (const int32_t*)a1;
  P.lval = (const double*)a2;
  P.ucol = (const int32_t*)a3;
  P.uval = (const double*)a4;
  P.ford = (const int32_t*)a5;
  P.bord = (const int32_t*)a6;
  P.rflag = (unsigned int*)a7;
  P.ntiles = nlev;  // (diagnostic: level count)
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ilu_csr<false>, 256, 0);
  const int64_t cap = (int64_t)(occ < 1 ? 1 : occ) * h->num_sm;
  const int64_t need = (n + 255) / 256;
  h->ilu_grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
  return PBICG_OK;
}

// stencil rows of this rank written out as CSR (global columns, ascending; Dirichlet
// legs dropped) for the ILU(0) handles, which run the CSR schedule
void stencil_rows_csr(const pbicg_stencil* op, int64_t row_begin, int64_t n_local,
                      std::vector<int64_t>* rp, std::vector<int32_t>* ci, std::vector<double>* va) {
  const int64_t nx = op->nx, ny = op->ny, nz = op->dim == 3 ? op->nz : 1;
  const int64_t pxy = nx * ny;
  const double* c = op->coef;
  rp->assign((size_t)n_local + 1, 0);
  ci->clear();
  va->clear();
  for (int64_t r = 0; r < n_local; ++r) {
    const int64_t row = row_begin + r;
    const int64_t x = row % nx, y = (row / nx) % ny, z = row / pxy;
    auto put = [&](int64_t col, double v) { ci->push_back((int32_t)col); va->push_back(v); };
    if (op->dim == 3 && z > 0) put(row - pxy, c[5]);
    if (y > 0) put(row - nx, c[3]);
    if (x > 0) put(row - 1, c[1]);
    put(row, c[0]);
    if (x < nx - 1) put(row + 1, c[2]);
    if (y < ny - 1) put(row + nx, c[4]);
    if (op->dim == 3 && z < nz - 1) put(row + pxy, c[6]);
    (*rp)[(size_t)r + 1] = (int64_t)ci->size();
  }
}

void destroy_one(pbicg_ctx* h) {
  if (h->stream) cudaStreamSynchronize(h->stream);
  collect_timing(h);
  destroy_graphs(h);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : h->allocs) cudaFree(p);
  if (h->scal_host) cudaFreeHost(h->scal_host);
  cudaEvent_t evs[] = {h->ev_entry, h->ev_poll[0], h->ev_poll[1], h->ev_fork, h->ev_join};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->comm == COMM_NCCL && nccl_api().ok) {
    if (h->nccl_red && h->nccl_red != h->nccl_halo) nccl_api().CommDestroy(h->nccl_red);
    if (h->nccl_halo) nccl_api().CommDestroy(h->nccl_halo);
  }
  bool own_stream = h->own_stream;
  cudaStream_t s = h->stream;
  if (pbicg_group* grp = h->group) {
    // the group's shared stream is destroyed with its last member
    for (auto& m : grp->m)
      if (m == h) m = nullptr;
    grp->alive--;
    if (own_stream && grp->alive > 0) {
      for (auto& m : grp->m)
        if (m) {
          m->own_stream = true;
          own_stream = false;
          break;
        }
    }
    if (grp->alive == 0) delete grp;
  }
  if (own_stream && s) cudaStreamDestroy(s);
  cudaGetLastError();
  delete h;
}

// ------------------------------- solve ----------------------------------------
struct SolveArgs {
  const double* b;
  const double* x0;
  double* x;
};

pbicg_status solve_members(const Members& G, const std::vector<SolveArgs>& io, double tol,
                           int32_t maxit, int32_t rr_period, double* rnorm_hist, double* gap_hist,
                           int32_t* iters_out, int32_t* outcome_out) {
  pbicg_ctx* h = G[0];
  for (pbicg_ctx* m : G)
    if (m->failed) return fail(h, PBICG_ESTATE, "handle is in a failed state");
  if (!rnorm_hist || !iters_out || !outcome_out) return fail(h, PBICG_EINVAL, "NULL argument");
  if (maxit < 0 || rr_period < 0 || !(tol >= 0.0))
    return fail(h, PBICG_EINVAL, "maxit, rr_period and tol must be >= 0");
  if (h->method != M_PBICGSTAB && rr_period != 0)
    return fail(h, PBICG_EINVAL, "residual replacement is defined for p-BiCGStab only (method 0)");
  if (h->auto_rr && rr_period != 0)
    return fail(h, PBICG_EINVAL, "rr_period must be 0 with automated replacement (rr_auto)");
  for (size_t r = 0; r < G.size(); ++r) {
    if (!io[r].b || !io[r].x0 || !io[r].x) return fail(h, PBICG_EINVAL, "NULL vector argument");
    ST(ensure_hist(G[r], (int64_t)maxit + 1));
  }
  ST(entry_sync(h));
  for (size_t r = 0; r < G.size(); ++r) {
    pbicg_ctx* m = G[r];
    m->gap_on = gap_hist != nullptr;
    const size_t nb = (size_t)m->n_local * sizeof(double);
    CU(cudaMemcpyAsync(m->V.b, io[r].b, nb, cudaMemcpyDeviceToDevice, m->stream));
    CU(cudaMemcpyAsync(m->V.x, io[r].x0, nb, cudaMemcpyDeviceToDevice, m->stream));
    // A1: g, s, l, z_{-1} (and the spare buffers) start at zero
    // (ILU(0): n_{-1} = M^-1 z_{-1} = 0 is read from nv by the first sweep A)
    double* zs[] = {m->V.g, m->V.s, m->V.l, m->V.z0, m->V.z1, m->V.zrr, m->ilu ? m->V.nv : nullptr};
    for (double* v : zs)
      if (v) CU(cudaMemsetAsync(v - m->H, 0, nb + 2 * m->H * sizeof(double), m->stream));
    Scal s0;
    memset(&s0, 0, sizeof(s0));
    s0.tol = tol;
    s0.sqrt_eps = std::sqrt(std::ldexp(1.0, -53));
    s0.outcome = OUT_MAXIT;
    s0.gap_iter = -1;
    s0.bench = m->bench;
    s0.rr_period = rr_period;
    s0.method = m->method;
    s0.auto_rr = m->auto_rr;
    s0.p2p = m->p2p;
    if (m->p2p) {
      s0.p2p_epoch = m->p2p_ep;
      for (int q = 0; q < m->nranks; ++q) {
        s0.p2p_recv[q] = m->p2p_recv_tab[q];
        s0.p2p_flag[q] = m->p2p_flag_tab[q];
      }
    }
    s0.ar_nA = m->ar_nA;
    s0.ar_muN = m->ar_muN;
    s0.ar_mutN = m->ar_mutN;
    s0.ar_eps = std::ldexp(1.0, -53);
    s0.ar_tau = std::sqrt(s0.ar_eps);
    s0.nranks = m->nranks;
    s0.rank = m->rank;
    s0.dist = m->dist;
    s0.red_send = m->red_send;
    s0.red_recv = m->red_recv;
    m->scal_host[0] = s0;
    CU(cudaMemcpyAsync(m->scal, m->scal_host, sizeof(Scal), cudaMemcpyHostToDevice, m->stream));
  }
  enq_init(G);
  CU(cudaGetLastError());
  // chunk length: even (double-buffer parity) and a multiple of the replacement
  // period so every chunk has the same replacement pattern (A11)
  const int P = rr_period;
  int L = 32;
  if (P > 0) {
    L = P;
    while (L < 32 || (L & 1)) L += P;
  }
  int64_t done_its = 0;
  int slot = 0;
  bool have_prev = false, stop = false;
  while (done_its < maxit && !stop) {
    const int n = (int)((maxit - done_its) < L ? (maxit - done_its) : L);
    pbicg_status st = run_chunk(G, n, P);
    if (st) {
      for (pbicg_ctx* m : G) m->failed = true;
      return st;
    }
    done_its += n;
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
  const Scal S = h->scal_host[0];
  int32_t iters = S.done ? S.iters : S.iter;
  if (iters > maxit) iters = maxit;
  if (iters < 0) iters = 0;
  CU(cudaMemcpy(rnorm_hist, h->hist.rnorm, (size_t)(iters + 1) * sizeof(double),
                cudaMemcpyDeviceToHost));
  if (gap_hist)
    CU(cudaMemcpy(gap_hist, h->hist.gap, (size_t)(iters + 1) * sizeof(double),
                  cudaMemcpyDeviceToHost));
  for (size_t r = 0; r < G.size(); ++r) {
    pbicg_ctx* m = G[r];
    CU(cudaMemcpyAsync(io[r].x, m->V.x, (size_t)m->n_local * sizeof(double),
                       cudaMemcpyDeviceToDevice, m->stream));
  }
  CU(cudaStreamSynchronize(h->stream));
  for (pbicg_ctx* m : G)
    if (m->timing) collect_timing(m);
  *iters_out = iters;
  *outcome_out = S.done ? S.outcome : OUT_MAXIT;
  for (pbicg_ctx* m : G) m->last_iters = iters;
  h->last_nrr = S.n_rr;
  return PBICG_OK;
}

// NCCL ranks: the automated-replacement constants by the rank chain of
// csr_bound_chain_step (window of partial column sums rank r -> r + 1 over the halo
// communicator, then the exact all-gather of the four per-rank maxima)
pbicg_status csr_bound_nccl(pbicg_ctx* h, const pbicg_csr* op, int bj) {
  const int64_t H = h->H;
  const int P = h->nranks, r = h->rank;
  auto& api = nccl_api();
  void *dwin = nullptr, *dparts = nullptr;
  ST(dalloc(h, &dwin, (size_t)2 * H * sizeof(double)));
  ST(dalloc(h, &dparts, (size_t)4 * P * sizeof(double)));
  std::vector<double> win_in((size_t)2 * H), win_out((size_t)2 * H), parts((size_t)4 * P, 0.0);
  if (r > 0) {
    NC(api.Recv(dwin, (size_t)2 * H, ncclDouble, r - 1, h->nccl_halo, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaMemcpy(win_in.data(), dwin, (size_t)2 * H * sizeof(double), cudaMemcpyDeviceToHost));
  }
  csr_bound_chain_step(op, bj, H, r == P - 1, r > 0 ? win_in.data() : nullptr,
                       r + 1 < P ? win_out.data() : nullptr, &parts[(size_t)4 * r]);
  if (r + 1 < P) {
    ST(upload(h, dwin, win_out.data(), (size_t)2 * H * sizeof(double)));
    NC(api.Send(dwin, (size_t)2 * H, ncclDouble, r + 1, h->nccl_halo, h->stream));
    CU(cudaStreamSynchronize(h->stream));
  }
  ST(upload(h, dparts, parts.data(), parts.size() * sizeof(double)));  // zero but row r
  NC(api.AllReduce(dparts, dparts, (size_t)4 * P, ncclDouble, ncclSum, h->nccl_halo, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  CU(cudaMemcpy(parts.data(), dparts, parts.size() * sizeof(double), cudaMemcpyDeviceToHost));
  bound_consts_from_parts(parts.data(), P, op->n_global, bj, &h->ar_nA, &h->ar_muN, &h->ar_mutN);
  h->ar_ok = true;
  return PBICG_OK;
}

// 0: not an incomplete factorisation; 1: ILU(0); 2: ICC(0) (reading A34)
int prec_ilu(int prec) {
  return prec == PBICG_PREC_ILU0 ? 1 : prec == PBICG_PREC_ICC0 ? 2 : 0;
}

// An ILU(0) / ICC(0) stencil handle runs the CSR schedule (stored n = M^-1 z and
// m = M^-1 w, the paper's split schedule) on the stencil written out as CSR for this
// rank's slab (ghost band = one plane / line), with the stencil wavefront kernels for
// M^-1 (the factors are those of the slab's diagonal block).
pbicg_status build_stencil_ilu(pbicg_ctx* h, const pbicg_stencil* op, int ilu) {
  if (ilu == 2 && (op->coef[1] != op->coef[2] || op->coef[3] != op->coef[4] ||
                   (op->dim == 3 && op->coef[5] != op->coef[6])))
    return fail(h, PBICG_EINVAL, "ICC(0) needs a symmetric stencil (use PBICG_PREC_ILU0)");
  const int64_t nz = op->dim == 3 ? op->nz : 1;
  const int64_t outer = op->dim == 3 ? nz : op->ny;
  const int64_t plane = op->dim == 3 ? op->nx * op->ny : op->nx;
  Geo& g = h->geo;
  g.nx = op->nx;
  g.ny = op->ny;
  g.nog = outer;
  slab(outer, h->nranks, h->rank, &g.o0, &g.nol);
  g.pxy = plane;
  for (int i = 0; i < 7; ++i) g.c[i] = op->coef[i];
  g.dinv = 1.0 / op->coef[0];
  h->dim = op->dim;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> va;
  const int64_t rb = g.o0 * plane, nl = g.nol * plane;
  stencil_rows_csr(op, rb, nl, &rp, &ci, &va);
  pbicg_csr c2{op->nx * op->ny * nz, rb, nl, rp.data(), ci.data(), va.data()};
  std::vector<double> dinv;
  int64_t width = 0;
  bool uniform = true;
  pbicg_status st = validate_csr(&c2, h->nranks, &dinv, &width, &uniform, plane);
  if (st) return fail(h, st, g_create_err);
  return build_csr(h, &c2, dinv, width, uniform, 1, ilu, op, plane);
}

// P handles sharing one stream (loopback transport)
pbicg_group* new_group(void* cuda_stream, cudaStream_t* s, bool* own) {
  *s = (cudaStream_t)cuda_stream;
  *own = false;
  if (!*s) {
    if (cudaStreamCreateWithFlags(s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    *own = true;
  }
  return new pbicg_group();
}

}  // namespace

// ===========================================================================
extern "C" {

pbicg_status pbicgstab_create_stencil(const pbicg_stencil* op, pbicg_prec prec,
                                      const pbicg_dist* dist, void* cuda_stream,
                                      pbicg_handle* out) {
  if (!out) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  *out = nullptr;
  const int ilu = prec_ilu(prec);
  const int bj = ilu ? 1 : prec_block(prec);
  if (!bj || bj > 8)
    return fail(nullptr, PBICG_EINVAL,
                "stencil prec must be PBICG_PREC_JACOBI, _ILU0, _ICC0 or PBICG_PREC_BJ(2|4|8)");
  const int nranks = dist ? dist->nranks : 1;
  if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
    return fail(nullptr, PBICG_EINVAL, "inconsistent nranks/rank");
  ST(validate_stencil(op, nranks));
  pbicg_ctx* h = new pbicg_ctx();
  h->nranks = nranks;
  h->rank = dist ? dist->rank : 0;
  pbicg_status st = common_setup(h, cuda_stream);
  if (!st && (nranks > 1 || (dist && dist->nccl_id_halo))) st = nccl_setup(h, dist);
  if (!st) st = ilu ? build_stencil_ilu(h, op, ilu) : build_stencil(h, op, bj);
  if (!st && ilu && h->dist) {  // dinv ghosts of the CSR schedule, once (collective)
    comm_halo(Members{h}, {[](pbicg_ctx* c) { return c->dinv_g; }});
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) st = fail(h, PBICG_ECUDA, cudaGetErrorString(e));
  }
  if (st) {
    g_create_err = h->err;
    destroy_one(h);
    return st;
  }
  *out = h;
  return PBICG_OK;
}

pbicg_status pbicgstab_create_csr(const pbicg_csr* op, pbicg_prec prec, const pbicg_dist* dist,
                                  void* cuda_stream, pbicg_handle* out) {
  if (!out) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  *out = nullptr;
  const int ilu = prec_ilu(prec);
  const int bj = ilu ? 1 : prec_block(prec);
  if (!bj)
    return fail(nullptr, PBICG_EINVAL,
                "prec must be PBICG_PREC_JACOBI, _ILU0, _ICC0 or PBICG_PREC_BJ(2..32)");
  if (ilu == 2 && op && op->row_ptr && !block_symmetric(op))
    return fail(nullptr, PBICG_EINVAL, "ICC(0) needs a symmetric (diagonal block of the) matrix");
  const int nranks = dist ? dist->nranks : 1;
  if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
    return fail(nullptr, PBICG_EINVAL, "inconsistent nranks/rank");
  std::vector<double> dinv;
  int64_t width = 0;
  bool uniform = true;
  ST(validate_csr(op, nranks, &dinv, &width, &uniform));
  pbicg_ctx* h = new pbicg_ctx();
  h->nranks = nranks;
  h->rank = dist ? dist->rank : 0;
  pbicg_status st = common_setup(h, cuda_stream);
  if (!st && (nranks > 1 || (dist && dist->nccl_id_halo))) st = nccl_setup(h, dist);
  if (!st) st = build_csr(h, op, dinv, width, uniform, bj, ilu);
  if (!st && h->comm == COMM_NCCL && nranks > 1 && !ilu) st = csr_bound_nccl(h, op, bj);
  if (!st && h->dist) {  // dinv ghosts, once (collective)
    comm_halo(Members{h}, {[](pbicg_ctx* c) { return c->dinv_g; }});
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) st = fail(h, PBICG_ECUDA, cudaGetErrorString(e));
  }
  if (st) {
    g_create_err = h->err;
    destroy_one(h);
    return st;
  }
  *out = h;
  return PBICG_OK;
}

pbicg_status pbicgstab_create_stencil_loopback(const pbicg_stencil* op, pbicg_prec prec,
                                               int32_t nranks, void* cuda_stream,
                                               pbicg_handle* out) {
  if (!out) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  const int ilu = prec_ilu(prec);
  const int bj = ilu ? 1 : prec_block(prec);
  if (!bj || bj > 8)
    return fail(nullptr, PBICG_EINVAL,
                "stencil prec must be PBICG_PREC_JACOBI, _ILU0, _ICC0 or PBICG_PREC_BJ(2|4|8)");
  ST(validate_stencil(op, nranks));
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  cudaStream_t s;
  bool own;
  pbicg_group* grp = new_group(cuda_stream, &s, &own);
  if (!grp) return fail(nullptr, PBICG_ECUDA, "stream creation failed");
  pbicg_status st = PBICG_OK;
  for (int r = 0; r < nranks && !st; ++r) {
    pbicg_ctx* h = new pbicg_ctx();
    h->nranks = nranks;
    h->rank = r;
    h->comm = COMM_LOOP;
    h->dist = nranks > 1;
    h->group = grp;
    grp->m.push_back(h);
    grp->alive++;
    st = common_setup(h, s);
    if (r == 0) h->own_stream = own;
    if (!st) st = ilu ? build_stencil_ilu(h, op, ilu) : build_stencil(h, op, bj);
    if (st) g_create_err = h->err;
  }
  if (!st && ilu && nranks > 1) {  // dinv ghosts of the CSR schedule
    comm_halo(grp->m, {[](pbicg_ctx* c) { return c->dinv_g; }});
    if (cudaStreamSynchronize(s) != cudaSuccess) st = fail(nullptr, PBICG_ECUDA, "dinv halo");
  }
  if (st) {
    Members m = grp->m;
    for (auto it = m.rbegin(); it != m.rend(); ++it) destroy_one(*it);
    return st;
  }
  for (int r = 0; r < nranks; ++r) out[r] = grp->m[r];
  return PBICG_OK;
}

pbicg_status pbicgstab_create_csr_loopback(const pbicg_csr* ops, pbicg_prec prec, int32_t nranks,
                                           void* cuda_stream, pbicg_handle* out) {
  if (!out || !ops || nranks < 1) return fail(nullptr, PBICG_EINVAL, "bad argument");
  const int ilu = prec_ilu(prec);
  const int bj = ilu ? 1 : prec_block(prec);
  if (!bj)
    return fail(nullptr, PBICG_EINVAL,
                "prec must be PBICG_PREC_JACOBI, _ILU0, _ICC0 or PBICG_PREC_BJ(2..32)");
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  std::vector<std::vector<double>> dinv(nranks);
  std::vector<int64_t> width(nranks);
  std::vector<char> uni(nranks);
  int64_t next = 0;
  for (int r = 0; r < nranks; ++r) {
    bool u = true;
    ST(validate_csr(&ops[r], nranks, &dinv[r], &width[r], &u));
    uni[r] = u;
    if (ops[r].row_begin != next || ops[r].n_global != ops[0].n_global)
      return fail(nullptr, PBICG_EINVAL, "rank row ranges must be contiguous and ordered");
    next += ops[r].n_local;
  }
  if (next != ops[0].n_global) return fail(nullptr, PBICG_EINVAL, "ranks must cover all rows");
  cudaStream_t s;
  bool own;
  pbicg_group* grp = new_group(cuda_stream, &s, &own);
  if (!grp) return fail(nullptr, PBICG_ECUDA, "stream creation failed");
  pbicg_status st = PBICG_OK;
  for (int r = 0; r < nranks && !st; ++r) {
    pbicg_ctx* h = new pbicg_ctx();
    h->nranks = nranks;
    h->rank = r;
    h->comm = COMM_LOOP;
    h->dist = nranks > 1;
    h->group = grp;
    grp->m.push_back(h);
    grp->alive++;
    st = common_setup(h, s);
    if (r == 0) h->own_stream = own;
    if (!st && ilu == 2 && !block_symmetric(&ops[r]))
      st = fail(h, PBICG_EINVAL, "ICC(0) needs symmetric diagonal blocks");
    if (!st) st = build_csr(h, &ops[r], dinv[r], width[r], uni[r] != 0, bj, ilu);
    if (st) g_create_err = h->err;
  }
  if (!st) {
    comm_halo(grp->m, {[](pbicg_ctx* c) { return c->dinv_g; }});
    if (cudaStreamSynchronize(s) != cudaSuccess) st = fail(nullptr, PBICG_ECUDA, "dinv halo");
  }
  if (!st) {
    double nA = 0, muN = 0, mutN = 0;
    // rank by rank, exactly as NCCL ranks do it (the window hand-over is a host copy)
    const int64_t H = PBICG_CSR_HALO;
    std::vector<double> parts((size_t)4 * nranks), win((size_t)2 * H), win2((size_t)2 * H);
    for (int r = 0; r < nranks; ++r) {
      csr_bound_chain_step(&ops[r], bj, H, r == nranks - 1, r > 0 ? win.data() : nullptr,
                           r + 1 < nranks ? win2.data() : nullptr, &parts[(size_t)4 * r]);
      win.swap(win2);
    }
    bound_consts_from_parts(parts.data(), nranks, ops[0].n_global, bj, &nA, &muN, &mutN);
    for (pbicg_ctx* m : grp->m) {
      m->ar_nA = nA;
      m->ar_muN = muN;
      m->ar_mutN = mutN;
      m->ar_ok = true;
    }
  }
  if (st) {
    Members m = grp->m;
    for (auto it = m.rbegin(); it != m.rend(); ++it) destroy_one(*it);
    return st;
  }
  for (int r = 0; r < nranks; ++r) out[r] = grp->m[r];
  return PBICG_OK;
}

pbicg_status pbicgstab_stencil_partition(const pbicg_stencil* op, int32_t nranks, int32_t rank,
                                         int64_t* row_begin, int64_t* n_local) {
  if (!row_begin || !n_local) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  if (rank < 0 || rank >= nranks) return fail(nullptr, PBICG_EINVAL, "inconsistent nranks/rank");
  ST(validate_stencil(op, nranks));
  const int64_t nz = op->dim == 3 ? op->nz : 1;
  const int64_t outer = op->dim == 3 ? nz : op->ny;
  const int64_t plane = op->dim == 3 ? op->nx * op->ny : op->nx;
  int64_t o0 = 0, nol = 0;
  slab(outer, nranks, rank, &o0, &nol);
  *row_begin = o0 * plane;
  *n_local = nol * plane;
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
  if (k == "transport") {  // collective for NCCL ranks; applies to every loopback member
    if (value < 0 || value > 1) return fail(h, PBICG_EINVAL, "transport must be 0 or 1");
    if (value == 1) {
      if (!h->dist)
        return fail(h, PBICG_EINVAL, "transport 1 needs several ranks (or an NCCL communicator)");
      ST(p2p_setup(members(h)));
    }
    for (pbicg_ctx* m : members(h)) {
      m->p2p = (int)value;
      set_peer_halo(m, value == 1);
      destroy_graphs(m);
    }
    return PBICG_OK;
  }
  for (pbicg_ctx* m : members(h)) {
    if (k == "bench") {
      m->bench = value != 0;
    } else if (k == "graphs") {
      m->use_graphs = value != 0;
    } else if (k == "timing") {
      m->timing = value != 0;
    } else if (k == "csr_tma") {  // CSR: TMA-staged sweeps (1, default) or per-row loads
      m->cst_on = value != 0;
      destroy_graphs(m);
    } else if (k == "pdl") {  // programmatic dependent launch of the tile kernels
      m->tg.pdl = value != 0;
      destroy_graphs(m);
    } else if (k == "overlap") {
      m->overlap = value != 0 && (m->comm != COMM_NCCL || m->nccl_red != m->nccl_halo);
      destroy_graphs(m);
    } else if (k == "tile") {
      if (value == 0 && m->kind == KIND_STENCIL && m->tg.bj > 1)
        return fail(h, PBICG_EINVAL, "block Jacobi on a stencil runs on the tile kernels only");
      m->tile_on = value != 0;
      destroy_graphs(m);
    } else if (k == "rr_auto") {
      if (value != 0 && m->ilu)
        return fail(h, PBICG_EINVAL, "rr_auto is not defined for ILU(0) / ICC(0) (reading A34)");
      if (value != 0 && (m->method != M_PBICGSTAB || !m->ar_ok ||
                         (m->kind == KIND_STENCIL && (!m->tile_ok || m->schedule == 2))))
        return fail(h, PBICG_EINVAL,
                    "rr_auto needs method 0 and a stencil on the TMA tile kernels (not odd nx > 1024) "
                    "or a CSR operator");
      m->auto_rr = value != 0;
      destroy_graphs(m);
    } else if (k == "method") {
      if (value != M_PBICGSTAB && m->auto_rr)
        return fail(h, PBICG_EINVAL, "switch rr_auto off before selecting method 1 or 2");
      if (value < 0 || value > 2) return fail(h, PBICG_EINVAL, "method must be 0, 1 or 2");
      if (value != M_PBICGSTAB && m->kind == KIND_STENCIL && m->schedule == 2)
        return fail(h, PBICG_EINVAL, "methods 1 and 2 run their own schedules (set schedule 0)");
      if (value != M_PBICGSTAB && m->kind == KIND_STENCIL && !m->tile_ok)
        return fail(h, PBICG_EINVAL,
                    "methods 1 (BiCGStab) and 2 (p-CG) on a stencil need nx <= 1024 "
                    "(TMA tile kernels)");
      m->method = (int)value;
      destroy_graphs(m);
    } else if (k == "schedule") {
      if (value < 0 || value > 2) return fail(h, PBICG_EINVAL, "schedule must be 0, 1 or 2");
      if (value == 2 && m->kind == KIND_STENCIL) {
        if (!m->tile_ok || m->tg.bj > 1 || m->auto_rr || m->method != M_PBICGSTAB)
          return fail(h, PBICG_EINVAL,
                      "split stencil schedule: Jacobi, nx <= 1024, method 0, rr_auto off");
        if (!m->V.tv) {
          ST(gvec(m, &m->V.tv));
          ST(gvec(m, &m->V.vv));
        }
      }
      if (value == 1 && m->kind == KIND_CSR)
        return fail(h, PBICG_EINVAL, "fused schedule is stencil-only");
      m->schedule = (int)value;
      destroy_graphs(m);
    } else {
      return fail(h, PBICG_EINVAL, "unknown option '" + k + "'");
    }
  }
  return PBICG_OK;
}

pbicg_status pbicgstab_apply(pbicg_handle h, const double* x_dev, double* y_dev) {
  if (!h || !x_dev || !y_dev) return fail(h, PBICG_EINVAL, "NULL argument");
  if (h->comm == COMM_LOOP) return fail(h, PBICG_EINVAL, "use pbicgstab_apply_loopback");
  ST(entry_sync(h));
  CU(cudaMemcpyAsync(h->xtmp, x_dev, (size_t)h->n_local * sizeof(double),
                     cudaMemcpyDeviceToDevice, h->stream));
  comm_halo(Members{h}, {[](pbicg_ctx* c) { return c->xtmp; }});
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

pbicg_status pbicgstab_apply_loopback(pbicg_handle* hs, int32_t nranks, const double* const* x_dev,
                                      double* const* y_dev) {
  if (!hs || nranks < 1 || !x_dev || !y_dev) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  pbicg_ctx* h = hs[0];
  if (!h || h->comm != COMM_LOOP || (int)h->group->m.size() != nranks)
    return fail(h, PBICG_EINVAL, "not a loopback group of this size");
  Members G = h->group->m;
  ST(entry_sync(h));
  for (int r = 0; r < nranks; ++r) {
    pbicg_ctx* m = G[r];
    CU(cudaMemcpyAsync(m->xtmp, x_dev[r], (size_t)m->n_local * sizeof(double),
                       cudaMemcpyDeviceToDevice, m->stream));
  }
  comm_halo(G, {[](pbicg_ctx* c) { return c->xtmp; }});
  for (int r = 0; r < nranks; ++r) {
    pbicg_ctx* m = G[r];
    LaunchScope ls(m, K_APPLY);
    if (m->kind == KIND_CSR)
      c_apply<<<m->grid[K_APPLY], m->block, 0, m->stream>>>(m->csr, m->xtmp, y_dev[r]);
    else if (m->dim == 3)
      k_apply<3><<<m->grid[K_APPLY], m->block, 0, m->stream>>>(m->geo, m->xtmp, y_dev[r]);
    else
      k_apply<2><<<m->grid[K_APPLY], m->block, 0, m->stream>>>(m->geo, m->xtmp, y_dev[r]);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->stream));
  return PBICG_OK;
}

pbicg_status pbicgstab_solve(pbicg_handle h, const double* b_dev, const double* x0_dev,
                             double tol, int32_t maxit, int32_t rr_period, double* x_dev_out,
                             double* rnorm_hist, double* gap_hist, int32_t* iters_out,
                             int32_t* outcome_out) {
  if (!h) return fail(nullptr, PBICG_EINVAL, "NULL handle");
  if (h->comm == COMM_LOOP) return fail(h, PBICG_EINVAL, "use pbicgstab_solve_loopback");
  std::vector<SolveArgs> io{{b_dev, x0_dev, x_dev_out}};
  return solve_members(Members{h}, io, tol, maxit, rr_period, rnorm_hist, gap_hist, iters_out,
                       outcome_out);
}

pbicg_status pbicgstab_solve_loopback(pbicg_handle* hs, int32_t nranks,
                                      const double* const* b_dev, const double* const* x0_dev,
                                      double tol, int32_t maxit, int32_t rr_period,
                                      double* const* x_dev_out, double* rnorm_hist,
                                      double* gap_hist, int32_t* iters_out,
                                      int32_t* outcome_out) {
  if (!hs || nranks < 1 || !b_dev || !x0_dev || !x_dev_out)
    return fail(nullptr, PBICG_EINVAL, "NULL argument");
  pbicg_ctx* h = hs[0];
  if (!h || h->comm != COMM_LOOP || (int)h->group->m.size() != nranks)
    return fail(h, PBICG_EINVAL, "not a loopback group of this size");
  std::vector<SolveArgs> io;
  for (int r = 0; r < nranks; ++r) io.push_back({b_dev[r], x0_dev[r], x_dev_out[r]});
  return solve_members(h->group->m, io, tol, maxit, rr_period, rnorm_hist, gap_hist, iters_out,
                       outcome_out);
}

pbicg_status pbicgstab_solve_host(pbicg_handle h, const double* b_host, const double* x0_host,
                                  double tol, int32_t maxit, int32_t rr_period,
                                  double* x_host_out, double* rnorm_hist, double* gap_hist,
                                  int32_t* iters_out, int32_t* outcome_out) {
  if (!h) return fail(nullptr, PBICG_EINVAL, "NULL handle");
  if (!b_host || !x0_host || !x_host_out) return fail(h, PBICG_EINVAL, "NULL argument");
  if (h->comm == COMM_LOOP) return fail(h, PBICG_EINVAL, "host entry is per process");
  const size_t nb = (size_t)h->n_local * sizeof(double);
  ST(entry_sync(h));
  // stage through the handle's own buffers: b -> V.rh (overwritten by init), x0 -> xtmp
  CU(cudaMemcpyAsync(h->xtmp, x0_host, nb, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(h->V.rh, b_host, nb, cudaMemcpyHostToDevice, h->stream));
  ST(pbicgstab_solve(h, h->V.rh, h->xtmp, tol, maxit, rr_period, h->xtmp, rnorm_hist, gap_hist,
                     iters_out, outcome_out));
  CU(cudaMemcpy(x_host_out, h->xtmp, nb, cudaMemcpyDeviceToHost));
  return PBICG_OK;
}

pbicg_status pbicgstab_kernel_time(pbicg_handle h, const char* name, int64_t* launches, double* ms,
                                   int32_t reset) {
  if (!h || !name) return fail(h, PBICG_EINVAL, "NULL argument");
  std::string n(name);
  if (n == "halo") {  // halo exchanges enqueued (not kernels of this library)
    if (launches) *launches = h->halo_ops;
    if (ms) *ms = NAN;
    if (reset) h->halo_ops = 0;
    return PBICG_OK;
  }
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
    for (int k = 0; k < K_N; ++k) {
      h->launches[k] = 0;
      h->ms[k] = 0;
    }
  }
  return PBICG_OK;
}

pbicg_status pbicgstab_kernel_bytes(pbicg_handle h, const char* name, double* bytes) {
  if (!h || !name || !bytes) return fail(h, PBICG_EINVAL, "NULL argument");
  std::string n(name);
  const double N = (double)h->n_local;
  double b = 0;
  if (split_sched(h)) {
    // split schedule (SURVEY 8(a)'s 32 passes)
    if (n == "sweepA") b = 13 * 8 * N;       // read k,g,l,s,r,w,z,t,v; write g,s,l,z
    else if (n == "sweepC") b = 15 * 8 * N;  // read x,g,k,l,r,s,r^,w,z,t,v; write x,r,k,w
    else if (n == "spmvB" || n == "spmvD") b = 2 * 8 * N;
    else if (n == "rr1") b = 7 * 8 * N;
    else if (n == "rr2") b = 5 * 8 * N;
    else if (n == "gap") b = 3 * 8 * N;
    else if (n == "apply") b = 2 * 8 * N;
    else if (n == "init") b = 4 * 8 * N;     // mean of init1 and init2 (the tile kernels)
    else if (n == "iteration") b = 32 * 8 * N;
  } else if (h->kind == KIND_STENCIL) {
    // fused schedule: every vector read / written once per launch
    if (n == "cl1") b = 6 * 8 * N;        // Alg. 1: read r,p,s,r^; write p,s
    else if (n == "cl2") b = 2 * 8 * N;   // read r,s
    else if (n == "cl3") b = 7 * 8 * N;   // read r,s,x,p,r^; write x,r
    else if (n == "pcg") b = 16 * 8 * N;  // p-CG: read w,z,q,s,p,x,r,u; write the same 8
    else if (n == "iteration" && h->method == M_BICGSTAB) b = 15 * 8 * N;
    else if (n == "iteration" && h->method == M_PIPECG) b = 16 * 8 * N;
    else if (n == "sweepA") b = 11 * 8 * N;  // read k,g,l,w,s,z,r; write g,s,l,z
    else if (n == "sweepC") b = 13 * 8 * N;  // read x,g,k,l,r,s,w,z,r^; write x,r,k,w
    // tile replacement step: read x,b,g,r^; write r,k,s,l / read k,l,r^; write w,z
    // (line kernels: read x,b,g; write r,k,s,l / read r,s,r^; write w,z)
    else if (n == "rr1") b = (tile_rr(h) ? 8 : 7) * 8 * N;
    else if (n == "rr2") b = 5 * 8 * N;
    else if (n == "gap") b = 3 * 8 * N;
    else if (n == "apply") b = 2 * 8 * N;
    else if (n == "init") b = 4 * 8 * N;     // mean of init1 (x,b -> r,r^,k) and init2 (r,r^ -> w)
    else if (n == "iteration") b = 24 * 8 * N;
  } else {
    const double slots = (double)h->csr.width;  // ELL width
    const double mat = 12.0 * slots * N;        // val (8) + col (4) per slot
    // the iteration's SpMVs: window kernel with 16-bit column offsets when banded
    const double matw = h->win_ok ? 10.0 * slots * N : mat;
    // block Jacobi: each kernel applying M^-1 reads its rows of the block inverse
    // instead of dinv (bj doubles instead of 1 per row)
    const double pb = h->csr.bj > 1 ? (h->csr.bj - 1) * 8.0 * N : 0.0;
    if (n == "sweepA") b = 15 * 8 * N + pb;  // read k,g,l,w,s,z,t,v,r,dinv; write g,s,l,z,n
    else if (h->method == M_BICGSTAB && n == "spmvB") b = matw + 3 * 8 * N;  // mv in; s out; r^
    else if (h->method == M_BICGSTAB && n == "spmvD") b = matw + 4 * 8 * N;  // nv in; y out; r, s
    else if (n == "spmvB" || n == "spmvD") b = matw + 2 * 8 * N;  // n|m in, out
    else if (n == "apply") b = mat + 2 * 8 * N;
    else if (n == "init") b = matw + 4 * 8 * N;  // mean of the two init SpMVs (x0 -> r,r^,k; k -> w,m)
    else if (n == "sweepC") b = 17 * 8 * N + pb;  // read x,g,k,l,r,s,w,z,t,v,r^,dinv; write x,r,k,w,m
    else if (n == "rr1") b = 2 * mat + 8 * 8 * N;
    else if (n == "rr2") b = 2 * mat + 7 * 8 * N;
    else if (n == "gap") b = matw + 3 * 8 * N;
    else if (n == "iteration" && h->method == M_BICGSTAB) b = 2 * matw + 2 * 8 * N + 24 * 8 * N;
    else if (n == "iteration" && h->method == M_PIPECG) b = matw + 21 * 8 * N;
    else if (n == "cl1") b = 6 * 8 * N;   // c_cl_p: read r,p,s,dinv; write p, M^-1 p
    else if (n == "cl2") b = 4 * 8 * N;   // c_cl_u: read r,s,dinv; write M^-1 q
    else if (n == "cl3") b = 9 * 8 * N;   // c_cl_x: read x,mv,nv,r,s,y,r^; write x,r
    else if (n == "pcg") b = 19 * 8 * N;  // c_pc: read n,z,q,s,p,x,r,u,w,dinv; write 9
    else if (n == "prec" && h->ilu)  // ILU(0) apply: forward (v, uinv in; out) + backward
      b = 6 * 8 * N + (h->ilu_st ? 0.0                     // (out, uinv in; out); stencil legs
                                  : 12.0 * (h->ilu_op.wl + h->ilu_op.wu) * N + 8.0 * N);  // CSR
    else if (n == "prec") b = 2 * 8 * N + pb + 8 * N;  // block Jacobi m = M^-1 w: w, binv rows; m
    else if (n == "iteration" && h->ilu && h->method == M_PIPECG) {
      double pr = 0;
      pbicgstab_kernel_bytes(h, "prec", &pr);
      b = matw + 21 * 8 * N + pr;
    } else if (n == "iteration" && h->ilu && h->method == M_BICGSTAB) {
      double pr = 0;
      pbicgstab_kernel_bytes(h, "prec", &pr);
      b = 2 * matw + 2 * 8 * N + 24 * 8 * N + 2 * pr;
    } else if (n == "iteration" && h->ilu) {
      double pr = 0;  // sweeps read m, n instead of dinv and write neither: same passes
      pbicgstab_kernel_bytes(h, "prec", &pr);
      b = 2 * matw + 36 * 8 * N + 2 * pr;
    } else if (n == "iteration") b = 2 * matw + 36 * 8 * N + 2 * pb;
  }
  *bytes = b;
  return PBICG_OK;
}

pbicg_status pbicgstab_rr_info(pbicg_handle h, double* fr_hist, int32_t* rr_iters, int32_t cap,
                               int32_t* n_rr) {
  if (!h || !n_rr || cap < 0) return fail(h, PBICG_EINVAL, "NULL argument");
  if (h->last_iters < 0) return fail(h, PBICG_ESTATE, "no solve has completed on this handle");
  if (h->comm == COMM_LOOP && h->group && h->group->m[0] != h)
    return fail(h, PBICG_EINVAL, "loopback group: ask rank 0's handle");
  const int32_t n = h->last_nrr;
  *n_rr = n;
  if (fr_hist) {
    if (h->auto_rr) {
      CU(cudaMemcpy(fr_hist, h->hist.fr, (size_t)(h->last_iters + 1) * sizeof(double),
                    cudaMemcpyDeviceToHost));
    } else {
      for (int32_t i = 0; i <= h->last_iters; ++i) fr_hist[i] = NAN;
    }
  }
  if (rr_iters && n > 0) {
    const int32_t c = n < cap ? n : cap;
    CU(cudaMemcpy(rr_iters, h->hist.rrl, (size_t)c * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  return PBICG_OK;
}

pbicg_status pbicgstab_scalar_trace(pbicg_handle h, double* out, int32_t cap) {
  if (!h || !out || cap < 0) return fail(h, PBICG_EINVAL, "NULL argument");
  if (h->last_iters < 0) return fail(h, PBICG_ESTATE, "no solve has completed on this handle");
  if (h->comm == COMM_LOOP && h->group && h->group->m[0] != h)
    return fail(h, PBICG_EINVAL, "loopback group: ask rank 0's handle");
  if (h->method != M_PBICGSTAB) return fail(h, PBICG_EINVAL, "scalar trace: method 0 only");
  const int32_t n = h->last_iters < cap ? h->last_iters : cap;
  if (n > 0) CU(cudaMemcpy(out, h->hist.sc, (size_t)n * SC_W * sizeof(double), cudaMemcpyDeviceToHost));
  return PBICG_OK;
}

pbicg_status pbicgstab_get_unique_id(void* out128) {
  if (!out128) return fail(nullptr, PBICG_EINVAL, "NULL argument");
  auto& api = nccl_api();
  if (!api.ok) return fail(nullptr, PBICG_ESTATE, api.err);
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, PBICG_ENCCL, api.GetErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return PBICG_OK;
}

const char* pbicgstab_last_error(pbicg_handle h) {
  return h ? h->err.c_str() : g_create_err.c_str();
}

void pbicgstab_destroy(pbicg_handle h) {
  if (!h) return;
  destroy_one(h);
}

}  // extern "C"
