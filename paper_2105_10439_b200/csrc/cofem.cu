// cofem.cu -- context, PCG driver and C ABI of the B200 CoFEM hot path.
//
// One context = one dense dictionary shard resident on one GPU plus the PCG
// workspace.  The PCG loop is driven from the host but never waits on the
// device inside a solve: every scalar (gamma, eta, delta) is derived on the
// device, kernels early-exit once the device status says "done", and the host
// only polls that status LAG steps behind the enqueue front.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cofem_b200.h"
#include <cuda.h>

#include <type_traits>

#include "kernels.cuh"
#include "nccl.h"
#include "dct.cuh"
#include "dct1024.cuh"
#include "dct1.cuh"
#include <cufft.h>
#include "ozaki.cuh"
#include "pcg.cuh"
#include "persistent.cuh"

using namespace cofem;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) return fail(COFEM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKR(x)              \
  do {                      \
    int r_ = (x);           \
    if (r_ != 0) return r_; \
  } while (0)

constexpr int LAG = 3;
constexpr int CONV_FFT_N = 1024;        // overlap-save block of the FP64 convolution path
constexpr int CONV_FFT_MAX_TAPS = 512;  // >= 513 outputs per block          // host status poll distance (steps)
constexpr int QCHUNK = 32;      // max columns per contraction launch
constexpr int64_t PAD = 256;    // Np, Dp multiples (tile sizes divide it)
constexpr int MAX_SPLITS = 32;  // split-K partial blocks per contraction

// ---- NCCL, bound at run time so the library loads without it -------------
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  // point-to-point (halo exchange of time-sharded convolutions)
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
};
NcclApi g_nccl;

// ---- cuFFT, bound at run time (only the 1-D subsampled DCT uses it) --------
struct CufftApi {
  bool tried = false, ok = false;
  cufftResult (*planMany)(cufftHandle*, int, int*, int*, int, int, int*, int, int, cufftType, int) = nullptr;
  cufftResult (*execZ2Z)(cufftHandle, cufftDoubleComplex*, cufftDoubleComplex*, int) = nullptr;
  cufftResult (*setStream)(cufftHandle, cudaStream_t) = nullptr;
  cufftResult (*destroy)(cufftHandle) = nullptr;
};
CufftApi g_cufft;

int cufft_load() {
  if (g_cufft.tried) return g_cufft.ok ? 0 : fail(COFEM_ECUDA, "libcufft.so.11 not loadable");
  g_cufft.tried = true;
  const char* names[] = {"libcufft.so.11", "libcufft.so", "/usr/local/cuda/lib64/libcufft.so.11"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return fail(COFEM_ECUDA, std::string("dlopen libcufft.so.11 failed: ") + dlerror());
  g_cufft.planMany = (decltype(g_cufft.planMany))dlsym(h, "cufftPlanMany");
  g_cufft.execZ2Z = (decltype(g_cufft.execZ2Z))dlsym(h, "cufftExecZ2Z");
  g_cufft.setStream = (decltype(g_cufft.setStream))dlsym(h, "cufftSetStream");
  g_cufft.destroy = (decltype(g_cufft.destroy))dlsym(h, "cufftDestroy");
  g_cufft.ok = g_cufft.planMany && g_cufft.execZ2Z && g_cufft.setStream && g_cufft.destroy;
  return g_cufft.ok ? 0 : fail(COFEM_ECUDA, "libcufft missing symbols");
}

int nccl_load() {
  if (g_nccl.tried) return g_nccl.ok ? 0 : fail(COFEM_ENCCL, "libnccl.so.2 not loadable");
  g_nccl.tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return fail(COFEM_ENCCL, std::string("dlopen libnccl.so.2 failed: ") + dlerror());
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.errStr = (decltype(g_nccl.errStr))dlsym(h, "ncclGetErrorString");
  g_nccl.send = (decltype(g_nccl.send))dlsym(h, "ncclSend");
  g_nccl.recv = (decltype(g_nccl.recv))dlsym(h, "ncclRecv");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.allReduce && g_nccl.commDestroy;
  return g_nccl.ok ? 0 : fail(COFEM_ENCCL, "libnccl missing symbols");
}

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// A kernel's raised dynamic shared-memory limit is a per-device setting: the
// flags that avoid re-issuing cudaFuncSetAttribute are kept per device (and
// atomic: rank threads of an in-process shard group set them concurrently).
constexpr int MAX_DEVICES = 64;
struct DeviceFlags {
  std::atomic<bool> set[MAX_DEVICES] = {};
};
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= MAX_DEVICES ? 0 : d;
}
// raise `fn`'s dynamic shared memory limit to `bytes` once per device
template <typename F>
int smem_attr_once(DeviceFlags& flags, F* fn, size_t bytes) {
  const int dev = current_device();
  if (flags.set[dev].load(std::memory_order_acquire)) return 0;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return fail(COFEM_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  flags.set[dev].store(true, std::memory_order_release);
  return 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

int encode_u8_3d(CUtensorMap* m, void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                 uint32_t b2) {
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return fail(COFEM_ECUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = (EncodeTiledFn)fn;
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0, d0 * d1};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ptr, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COFEM_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return 0;
}

// K-blocked operand planes [k_pad / 64][4][ncols][64] (oz::kb_offset), box {64, box_cols, 4, 1}
int encode_u8_kblocked(CUtensorMap* m, void* ptr, uint64_t k_pad, uint64_t ncols, uint32_t box_cols) {
  if (!g_encode) {
    int rc = encode_u8_3d(m, ptr, 64, 8, 1, 64, 8, 1);  // resolves the driver entry point
    if (rc) return rc;
  }
  cuuint64_t dims[4] = {64, ncols, 4, k_pad / 64};
  cuuint64_t strides[3] = {64, 64 * ncols, 256 * ncols};
  cuuint32_t box[4] = {64, box_cols, 4, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, ptr, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COFEM_ECUDA, "cuTensorMapEncodeTiled (4d) failed: " + std::to_string((int)r));
  return 0;
}

// ---- contraction configurations -------------------------------------------
// fp32: 4 rows (fwd) / 4 columns (bwd) x QP accumulators per thread
// fp64: 2 x QP double accumulators per thread
template <typename T>
struct Tiles;
template <>
struct Tiles<float> {
  static constexpr int FR = 4, FWM = 2, FWK = 4, FBK = 32, FST = 2;
  static constexpr int BC = 4, BWN = 2, BWK = 4, BBK = 32, BST = 3;
};
template <>
struct Tiles<double> {
  static constexpr int FR = 2, FWM = 4, FWK = 2, FBK = 32, FST = 2;
  static constexpr int BC = 2, BWN = 4, BWK = 2, BBK = 32, BST = 2;
};

}  // namespace

struct SplitPlan {
  int nsplit = 1;
  int per_split = 0;  // rows (bwd) or columns (fwd) per split, multiple of the tile depth
};

// In-process shard group: the ranks of one sharded problem driven from host
// threads of ONE process (one context per rank, on one or several devices).
// It implements the same exchanges as the NCCL communicator -- all-reduce
// (sum / max) and the neighbour halo send/recv -- with stream-ordered events:
// a rank records "ready" after producing its buffer, a host barrier publishes
// the buffers, every rank's stream waits on the peers' events and reads the
// peers' buffers directly (device or peer memory), then a second event /
// barrier round keeps a buffer alive until every peer has read it.  No kernel
// ever waits on another rank's kernel.
struct cofem_group {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<void*> bufs;
  std::vector<cudaEvent_t> ready, done;
};

struct cofem_ctx {
  int device = 0, prec = COFEM_FP32;
  int64_t N = 0, D = 0, Np = 0, Dp = 0;
  int64_t col_offset = 0, global_cols = 0;
  // reference probe stream (cofem_set_probe_stream): PCG64 state before the
  // first draw; EM iteration t draws raw outputs [t ceil(D K / 2), ...)
  bool pcg_stream = false;
  uint64_t pcg_state[2] = {0, 0}, pcg_inc[2] = {0, 0};
  uint64_t pcg_first = 0, pcg_stride = 0;  // halves before draw 0; halves between iterations (0: D K)
  cudaStream_t stream = nullptr;
  float* phi = nullptr;
  double* phi64 = nullptr;  // exact float64 dictionary (fp64 mode, cofem_set_dictionary_f64)
  bool have_phi = false;
  int sm_count = 148;

  // workspace (T = float or double by precision)
  int ldq = 0;
  void *X = nullptr, *R = nullptr, *P = nullptr, *Psi = nullptr;
  void* P2 = nullptr;  // the other direction buffer (k_direction writes P(u+1) there; swapped per step)
  void *V = nullptr, *vpart = nullptr, *ppart = nullptr, *tmpD = nullptr;
  size_t vpart_cap = 0, ppart_cap = 0;
  double *alpha = nullptr, *minv = nullptr, *theta = nullptr, *colsq = nullptr;
  double *mu = nullptr, *s = nullptr, *aty = nullptr, *ybuf = nullptr;
  int8_t *probes = nullptr, *probe_store = nullptr;
  int* groups = nullptr;
  int groups_cap = 0;
  double* scal = nullptr;  // rho0 | rho1 | rho_new | rn2 | pi | bn2 | gam0 | gam1 | vv | pap (ldq each)
  int* frozen = nullptr;
  double* partials = nullptr;
  unsigned* tickets = nullptr;
  Status* st = nullptr;
  Status* h_st = nullptr;  // pinned + mapped, LAG slots (k_direction writes them)
  Status* d_hst = nullptr; // device alias of h_st
  cudaEvent_t ev[LAG] = {};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int nblk_elem = 0;

  // Ozaki (int8 tensor-core) contraction state
  bool oz_ready = false;
  int8_t* phiq = nullptr;        // [npa][Np][Dp] signed digit planes
  int npa = 4;                   // digit planes of Phi: 4 (32-bit fixed point) or 3 (24-bit, COFEM_OZAKI24)
  int8_t* phiqT = nullptr;       // [4][Dp][Np] the same planes transposed: Phi^T V streams K-major too
  CUtensorMap map_phiT{};
  double *rowscale = nullptr, *colscale = nullptr;  // Np, Dp powers of two
  int8_t *pq = nullptr, *vq = nullptr;              // operand planes, K-blocked [Dp/64][4][QW][64] / [Np/64][...]
  double* opscale = nullptr;                        // QCHUNK column scales
  unsigned long long* colmax = nullptr;             // P column maxima (up to 1024 columns)
  unsigned long long* vcolmax = nullptr;            // V column maxima (QCHUNK)
  bool p_colmax_valid = false, v_colmax_valid = false;
  CUtensorMap map_phi_fwd{}, map_phi_bwd{};
  CUtensorMap map_p[5]{}, map_v[5]{};               // by QW / 8
  bool map_p_ok[5] = {}, map_v_ok[5] = {};

  // operator kind: dense dictionary or banded Toeplitz convolution
  int kind = 0;                                      // 0 dense, 1 convolution
  int conv_L = 0, conv_lpad = 0;                     // taps, taps-1 rounded up to 64
  int8_t *band_fwd = nullptr, *band_adj = nullptr;   // [4][128][128 + lpad] digit planes
  double* hrows = nullptr;                           // Dp copies of the band's power-of-two scale
  std::vector<double> taps;                          // host copy (column norms of a time shard)
  CUtensorMap map_band_fwd{}, map_band_adj{};
  // float64 FFT path (precision FP64, <= 512 taps): overlap-save spectra of h
  // and of reversed h (1024 points, 1/1024 folded in); FFT twiddles in dct_wN
  bool conv_fft = false;
  double2 *cf_H = nullptr, *cf_Hr = nullptr;

  // 2-D partial DCT (kind 2): n x n images, D = n^2, N = mask size
  int dct_n = 0;
  int64_t* dct_mask = nullptr;      // N flat coefficient indices k n + l
  uint8_t* dct_grid = nullptr;      // n x n 0/1 mask grid [k][l]
  uint8_t* dct_gridT = nullptr;     // its transpose [l][k] (the column pass reads one l at a time)
  double *bufA = nullptr, *bufB = nullptr;  // n x n ldq pass buffers
  double2 *dct_wN = nullptr, *dct_tw = nullptr;  // e^{-2 pi i j / n}, e^{-i pi k / 2n} / sqrt(2n)
  // n = 1024 warp-per-FFT passes (dct1024.cuh): lane-contiguous step twiddles and the pair-mask bytes
  double2* dct_twF = nullptr;
  double2* dct_wT = nullptr;
  // Psi-free DCT step: vv | <P, alpha P> (VV_MAXQ each) and the last row pass's per-block partial sums
  double *dct_fscal = nullptr, *dct_partials = nullptr, *dct_partials4 = nullptr;
  int dct_vv_blocks = 0;  // step twiddles of the N1 x N2 four-step FFT, [k2][lt] = w_n^{lt k2}
  uint8_t* dct_pm = nullptr;
  double* dct_cn = nullptr;                      // orthonormal DCT-II scales c_k

  // 1-D subsampled DCT (kind 3, dct1.cuh): length D = N_cols, N = mask size;
  // dct_mask holds the sorted mask, bufA the complex [D][ldq / 2] work block
  uint8_t* dct1_mv = nullptr;  // the mask in Makhoul (v) order: mask[sigma(m)]
  cufftHandle fft_plan = 0;
  int fft_plan_hc = 0;         // column pairs the plan was made for (0: none)

  // multi-GPU
  ncclComm_t comm = nullptr;
  cofem_group* lgroup = nullptr;  // in-process shard group (instead of comm)
  void* lg_tmp = nullptr;         // its all-reduce result staging
  size_t lg_tmp_cap = 0;
  int nranks = 1, rank = 0;
  // time-sharded convolution: operand planes carry the neighbours' halo rows
  // (pq: conv_lpad rows before the data for rank > 0; vq: after it for rank < nranks-1)
  int8_t* pq_base = nullptr;

  // the last cofem_run: per-iteration wall times, probes K, final CG report
  std::vector<double> run_wall;
  int run_K = 0;
  cofem_cg_report run_rep{};

  // bench state
  bool bench_ready = false;
  double beta = 0;
  cofem_em_config em{};
  cofem_cg_config cg{};
  uint64_t dseed = 0;
  int bench_iter = 0;

  // persistent (one-launch) PCG solves: grid barrier words, phase stamps
  unsigned* gbar = nullptr;
  size_t gbar_cap = 0;
  unsigned long long* ptimes = nullptr;
  int ptimes_cap = 0;
  bool persistent_off = false;  // COFEM_NO_PERSISTENT: always the multi-kernel step
  bool conv_fused_off = false;  // COFEM_CONV_UNFUSED: the convolution step as separate quantise / update launches
  unsigned long long* fz_max = nullptr;  // fused convolution step: |P| maxima [2][32] (by step parity), |M^-1 R| [32]
  double ph_fwd_ms = 0, ph_bwd_ms = 0, solve_ms = 0;
  int64_t solve_launches = 0;

  // instrumentation
  bool time_kernels = false;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  std::vector<std::pair<int, size_t>> timed;  // (kind 0 fwd / 1 bwd, event index)
  // COFEM_TICKS (bench runs): an event after every kernel of the 2-D DCT PCG step; (segment id, event before, event after)
  bool ticks_on = false;
  long tick_prev = -1;
  std::vector<std::array<long, 3>> ticks;
  int64_t launches = 0, fwd_launches = 0, bwd_launches = 0, pcg_steps = 0;

  Scalars sc() const {
    Scalars s;
    s.rho[0] = scal;
    s.rho[1] = scal + ldq;
    s.rho_new = scal + 2 * ldq;
    s.rn2 = scal + 3 * ldq;
    s.pi = scal + 4 * ldq;
    s.bn2 = scal + 5 * ldq;
    s.gam[0] = scal + 6 * ldq;
    s.gam[1] = scal + 7 * ldq;
    s.frozen = frozen;
    s.partials = partials;
    s.ticket = tickets;
    s.rev_rows = kind == 2 ? 1 : 0;
    return s;
  }
  size_t tsize() const { return prec == COFEM_FP32 ? 4 : 8; }
};

namespace {

int set_dev(cofem_ctx* c) {
  CK(cudaSetDevice(c->device));
  return 0;
}

// Host -> device copy ordered on the context stream, complete on return.
// (A plain cudaMemcpy runs on the legacy default stream, which does not order
// against the non-blocking context stream, and from pageable memory it may
// return before its DMA lands: kernels on the context stream could then read
// the old contents.)
cudaError_t h2d_sync(cofem_ctx* c, void* dst, const void* src, size_t bytes) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(c->stream);
}

cudaEvent_t next_event(cofem_ctx* c) {
  if (c->evnext == c->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evpool.push_back(e);
  }
  return c->evpool[c->evnext++];
}

// live per-kernel timing of a PCG step (COFEM_TICKS=1 with cofem_bench_iterations(time_kernels)):
// the segment since the previous tick is charged to `id`; id < 0 only restarts the chain
void tick(cofem_ctx* c, int id) {
  if (!c->ticks_on) return;
  cudaEvent_t e = next_event(c);
  cudaEventRecord(e, c->stream);
  const long cur = (long)c->evnext - 1;
  if (id >= 0 && c->tick_prev >= 0) c->ticks.push_back({(long)id, c->tick_prev, cur});
  c->tick_prev = cur;
}

void free_ws(cofem_ctx* c) {
  void* ptrs[] = {c->X, c->R, c->P, c->P2, c->Psi, c->V, c->vpart, c->ppart, c->tmpD, c->scal, c->frozen, c->partials};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  c->X = c->R = c->P = c->P2 = c->Psi = c->V = c->vpart = c->ppart = c->tmpD = nullptr;
  c->scal = nullptr;
  c->frozen = nullptr;
  c->partials = nullptr;
  c->ldq = 0;
}

// column-block kernels: blockDim a multiple of ldq near 512 (few blocks -> a
// short deterministic final reduction; 4 rows per thread trip for MLP)
int elem_block(int ldq) { return ldq >= 256 ? ldq : ldq * (256 / ldq); }  // 3 blocks / SM resident (<= 85 regs)

// choose split count for a contraction: minimise wave quantisation plus the
// extra traffic of the split partials relative to the Phi stream
SplitPlan plan_splits(int64_t nblocks_other, int64_t ntiles, int tile, int slots, double out_bytes_per_split,
                      double phi_bytes) {
  SplitPlan best;
  double best_cost = 1e300;
  const int smax = (int)std::min<int64_t>(ntiles, MAX_SPLITS);
  for (int s = 1; s <= smax; ++s) {
    const int64_t per = (ntiles + s - 1) / s;
    const int64_t S = (ntiles + per - 1) / per;
    const int64_t ctas = nblocks_other * S;
    const double waves = std::ceil((double)ctas / slots);
    const double t_compute = waves * per / ((double)nblocks_other * ntiles / slots);
    const double t_part = 2.0 * S * out_bytes_per_split / phi_bytes;
    const double cost = t_compute + t_part;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best.nsplit = (int)S;
      best.per_split = (int)(per * tile);
    }
  }
  return best;
}

// CUDA-core contractions over a float32 (PhiT = float) or exact float64
// (PhiT = double, fp64 mode) dictionary
template <typename T, int QP, typename PhiT = float>
struct Kern {
  using TL = Tiles<T>;
  using FC = FwdCfg<T, QP, TL::FR, TL::FWM, TL::FWK, TL::FBK, TL::FST, PhiT>;
  using BC = BwdCfg<T, QP, TL::BC, TL::BWN, TL::BWK, TL::BBK, TL::BST, PhiT>;
  static constexpr auto fwd = fwd_kernel<T, QP, TL::FR, TL::FWM, TL::FWK, TL::FBK, TL::FST, PhiT>;
  static constexpr auto bwd = bwd_kernel<T, QP, TL::BC, TL::BWN, TL::BWK, TL::BBK, TL::BST, PhiT>;
  static DeviceFlags flags;
  static std::atomic<int> fwd_occ, bwd_occ;  // same on every B200
  static int init() {
    const int dev = current_device();
    if (flags.set[dev].load(std::memory_order_acquire)) return 0;
    CK(cudaFuncSetAttribute(fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FC::SMEM));
    CK(cudaFuncSetAttribute(bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BC::SMEM));
    int fo = 0, bo = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fo, fwd, FC::NT, FC::SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bo, bwd, BC::NT, BC::SMEM));
    if (fo < 1 || bo < 1) return fail(COFEM_ECUDA, "contraction kernel cannot be resident");
    fwd_occ = fo;
    bwd_occ = bo;
    flags.set[dev].store(true, std::memory_order_release);
    return 0;
  }
};
template <typename T, int QP, typename PhiT>
DeviceFlags Kern<T, QP, PhiT>::flags;
template <typename T, int QP, typename PhiT>
std::atomic<int> Kern<T, QP, PhiT>::fwd_occ{0};
template <typename T, int QP, typename PhiT>
std::atomic<int> Kern<T, QP, PhiT>::bwd_occ{0};

int ensure_ws(cofem_ctx* c, int ldq) {
  if (c->ldq == ldq) return 0;
  free_ws(c);
  const size_t ts = c->tsize();
  const size_t dbytes = (size_t)c->Dp * ldq * ts;
  CK(cudaMalloc(&c->X, dbytes));
  CK(cudaMalloc(&c->R, dbytes));
  CK(cudaMalloc(&c->P, dbytes));
  CK(cudaMalloc(&c->P2, dbytes));
  CK(cudaMalloc(&c->Psi, dbytes));
  // the DCT passes transform all ldq columns at once; the contractions run
  // 32-column chunks
  const bool whole = c->kind == 2 || c->kind == 3 || c->conv_fft;  // passes over all ldq columns at once
  const int vcols = whole ? std::max(ldq, QCHUNK) : QCHUNK;
  CK(cudaMalloc(&c->tmpD, (size_t)c->Dp * vcols * ts));
  CK(cudaMalloc(&c->V, (size_t)c->Np * vcols * ts));
  // split partial capacity: up to MAX_SPLITS partial blocks of a 32-column
  // chunk for dense dictionaries; the banded operator writes one partial; the
  // DCT needs none
  const int max_splits = c->kind == 0 ? MAX_SPLITS : 1;
  c->vpart_cap = c->kind == 0 ? (size_t)max_splits * c->Np * QCHUNK * ts : 0;
  c->ppart_cap = whole ? 0 : (size_t)max_splits * c->Dp * QCHUNK * ts;
  if (c->vpart_cap) CK(cudaMalloc(&c->vpart, c->vpart_cap));
  if (c->ppart_cap) CK(cudaMalloc(&c->ppart, c->ppart_cap));
  CK(cudaMalloc(&c->scal, 10 * ldq * sizeof(double)));  // + vv | pap (fused convolution step)
  CK(cudaMalloc(&c->frozen, ldq * sizeof(int)));
  c->nblk_elem = 3 * c->sm_count;
  CK(cudaMalloc(&c->partials, (size_t)c->nblk_elem * 2 * std::max(ldq, QCHUNK) * sizeof(double)));
  CK(cudaMemsetAsync(c->X, 0, dbytes, c->stream));
  CK(cudaMemsetAsync(c->R, 0, dbytes, c->stream));
  CK(cudaMemsetAsync(c->P, 0, dbytes, c->stream));
  CK(cudaMemsetAsync(c->P2, 0, dbytes, c->stream));
  CK(cudaMemsetAsync(c->Psi, 0, dbytes, c->stream));
  if (c->kind == 3) {  // the complex [D][ldq / 2] work block
    if (c->bufA) cudaFree(c->bufA);
    CK(cudaMalloc(&c->bufA, (size_t)c->D * ldq * sizeof(double)));
  }
  if (c->kind == 2) {
    const int64_t n = c->dct_n, nc = n * ldq;
    for (double** b : {&c->bufA, &c->bufB}) {
      if (*b) cudaFree(*b);
      CK(cudaMalloc(b, (size_t)n * nc * sizeof(double)));
      CK(cudaMemsetAsync(*b, 0, (size_t)n * nc * sizeof(double), c->stream));
    }
  }
  c->ldq = ldq;
  return 0;
}

int ensure_groups(cofem_ctx* c, int n) {
  if (c->groups_cap >= n) return 0;
  if (c->groups) cudaFree(c->groups);
  CK(cudaMalloc(&c->groups, n * sizeof(int)));
  c->groups_cap = n;
  return 0;
}

// ---- exchanges: NCCL communicator or in-process shard group ---------------
int group_barrier(cofem_group* g) {
  std::unique_lock<std::mutex> lk(g->m);
  if (g->broken) return fail(COFEM_ENCCL, "shard group broken (a rank failed)");
  const uint64_t my = g->gen;
  if (++g->arrived == g->n) {
    g->arrived = 0;
    g->gen++;
    g->cv.notify_all();
    return 0;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(300), [&] { return g->gen != my || g->broken; })) {
    g->broken = true;
    g->cv.notify_all();
    return fail(COFEM_ENCCL, "shard group barrier timed out");
  }
  if (g->gen == my) return fail(COFEM_ENCCL, "shard group broken (a rank failed)");
  return 0;
}

void group_break(cofem_group* g) {
  if (!g) return;
  std::lock_guard<std::mutex> lk(g->m);
  g->broken = true;
  g->cv.notify_all();
}

// publish `mine`; run work(bufs) on c->stream once every rank's buffer is
// ready; return once every rank has finished reading this rank's buffer
template <class F>
int group_phase(cofem_ctx* c, void* mine, F&& work) {
  cofem_group* g = c->lgroup;
  const int r = c->rank;
  CK(cudaEventRecord(g->ready[r], c->stream));
  g->bufs[r] = mine;
  CKR(group_barrier(g));
  std::vector<void*> bufs(g->bufs);
  for (int i = 0; i < g->n; ++i)
    if (i != r) CK(cudaStreamWaitEvent(c->stream, g->ready[i], 0));
  int rc = work(bufs);
  if (rc) {
    group_break(g);
    return rc;
  }
  CK(cudaEventRecord(g->done[r], c->stream));
  CKR(group_barrier(g));
  for (int i = 0; i < g->n; ++i)
    if (i != r) CK(cudaStreamWaitEvent(c->stream, g->done[i], 0));
  return 0;
}

int group_allreduce(cofem_ctx* c, void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op) {
  const size_t es = dt == ncclFloat32 ? 4 : 8;
  if (dt != ncclFloat32 && dt != ncclFloat64 && dt != ncclUint64) return fail(COFEM_EINVAL, "group all-reduce type");
  if (c->lg_tmp_cap < count * es) {
    CK(cudaStreamSynchronize(c->stream));
    if (c->lg_tmp) cudaFree(c->lg_tmp);
    c->lg_tmp = nullptr;
    c->lg_tmp_cap = 0;
    CK(cudaMalloc(&c->lg_tmp, count * es));
    c->lg_tmp_cap = count * es;
  }
  const int mx = op == ncclMax ? 1 : 0;
  CKR(group_phase(c, buf, [&](std::vector<void*>& bufs) -> int {
    GroupPtrs gp{};
    for (int i = 0; i < c->nranks; ++i) gp.p[i] = bufs[i];
    const int grid = (int)std::min<size_t>((count + 255) / 256, 4 * (size_t)c->sm_count);
    if (dt == ncclFloat64) k_group_reduce<double><<<grid, 256, 0, c->stream>>>(gp, c->nranks, count, mx, (double*)c->lg_tmp);
    else if (dt == ncclFloat32) k_group_reduce<float><<<grid, 256, 0, c->stream>>>(gp, c->nranks, count, mx, (float*)c->lg_tmp);
    else k_group_reduce<unsigned long long><<<grid, 256, 0, c->stream>>>(gp, c->nranks, count, mx,
                                                                         (unsigned long long*)c->lg_tmp);
    c->launches++;
    CK(cudaGetLastError());
    return 0;
  }));
  CK(cudaMemcpyAsync(buf, c->lg_tmp, count * es, cudaMemcpyDeviceToDevice, c->stream));
  return 0;
}

int allreduce(cofem_ctx* c, void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op = ncclSum) {
  if (c->nranks <= 1) return 0;
  if (c->lgroup) return group_allreduce(c, buf, count, dt, op);
  if (!c->comm) return 0;
  ncclResult_t r = g_nccl.allReduce(buf, buf, count, dt, op, c->comm, c->stream);
  if (r != ncclSuccess) return fail(COFEM_ENCCL, std::string("ncclAllReduce: ") + (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
  return 0;
}

// neighbour exchange along the rank order: dir +1 sends `send` to rank+1 and
// receives `recv` from rank-1; dir -1 the reverse.  Ends of the chain keep
// their (zero) halo.
int halo_exchange(cofem_ctx* c, const void* send, void* recv, size_t bytes, int dir) {
  if (c->nranks <= 1) return 0;
  const int to = c->rank + dir, from = c->rank - dir;
  const bool has_to = to >= 0 && to < c->nranks, has_from = from >= 0 && from < c->nranks;
  if (c->lgroup) {
    return group_phase(c, const_cast<void*>(send), [&](std::vector<void*>& bufs) -> int {
      if (has_from) CK(cudaMemcpyAsync(recv, bufs[from], bytes, cudaMemcpyDefault, c->stream));
      return 0;
    });
  }
  if (!c->comm) return 0;
  if (!g_nccl.send || !g_nccl.recv || !g_nccl.groupStart || !g_nccl.groupEnd)
    return fail(COFEM_ENCCL, "libnccl lacks ncclSend / ncclRecv");
  ncclResult_t r = g_nccl.groupStart();
  if (r == ncclSuccess && has_to) r = g_nccl.send(send, bytes, ncclInt8, to, c->comm, c->stream);
  if (r == ncclSuccess && has_from) r = g_nccl.recv(recv, bytes, ncclInt8, from, c->comm, c->stream);
  ncclResult_t r2 = g_nccl.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return fail(COFEM_ENCCL, std::string("halo send/recv: ") + (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
  return 0;
}

// the all-reduce of a dense shard's partial Phi_r P_r; its column maxima are
// no longer those of the local partial
int reduce_partial_v(cofem_ctx* c, size_t count, ncclDataType_t dt) {
  if (c->kind != 0 || c->nranks <= 1) return 0;
  CKR(allreduce(c, c->V, count, dt));
  c->v_colmax_valid = false;
  return 0;
}

template <typename T>
ncclDataType_t nccl_t() {
  return sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
}

// ---- Ozaki int8 tensor-core contractions -----------------------------------
// digit planes + power-of-two scales of Phi; src = the dense float32 copy, or
// a float64 original (cofem_set_dictionary_f64) when given
int ensure_oz(cofem_ctx* c, const double* src64 = nullptr) {
  if (c->oz_ready && !src64) return 0;
  if (!c->phiq) {
    CK(cudaMalloc(&c->phiq, (size_t)c->npa * c->Np * c->Dp));
    CK(cudaMalloc(&c->rowscale, c->Np * sizeof(double)));
    CK(cudaMalloc(&c->colscale, c->Dp * sizeof(double)));
    CK(cudaMalloc(&c->pq, (size_t)4 * QCHUNK * c->Dp));
    CK(cudaMalloc(&c->vq, (size_t)4 * QCHUNK * c->Np));
    CK(cudaMalloc(&c->opscale, QCHUNK * sizeof(double)));
    CK(cudaMalloc(&c->colmax, 1024 * sizeof(unsigned long long)));
    CK(cudaMalloc(&c->vcolmax, QCHUNK * sizeof(unsigned long long)));
    CKR(encode_u8_3d(&c->map_phi_fwd, c->phiq, c->Dp, c->Np, c->npa, oz::KT, oz::BM, c->npa));
    CKR(encode_u8_3d(&c->map_phi_bwd, c->phiq, c->Dp, c->Np, c->npa, 64, oz::KT, c->npa));
    // COFEM_MN_MAJOR_ONLY: skip the transposed copy (Phi^T V reads the planes
    // MN-major) -- tests compare the two paths bitwise
    if (!getenv("COFEM_MN_MAJOR_ONLY") && cudaMalloc(&c->phiqT, (size_t)c->npa * c->Np * c->Dp) == cudaSuccess) {
      CKR(encode_u8_3d(&c->map_phiT, c->phiqT, c->Np, c->Dp, c->npa, oz::KT, oz::BM, c->npa));
    } else {
      cudaGetLastError();  // no room for the transposed copy: Phi^T V reads the planes MN-major
      c->phiqT = nullptr;
    }
  }
  // column shards agree on the row scales (max over every shard's columns),
  // so each shard's digit planes are the unsharded dictionary's columns and
  // every rank quantises the all-reduced V with the same scales
  const bool shard_rows = c->nranks > 1;
  auto row_scales = [&](auto* phi_src) -> int {
    using PT = std::remove_const_t<std::remove_pointer_t<decltype(phi_src)>>;
    oz::k_phi_rowscale<PT><<<(unsigned)c->Np, 256, 0, c->stream>>>(phi_src, c->Dp, c->N, c->D, c->rowscale,
                                                                    shard_rows);
    if (shard_rows) {
      CKR(allreduce(c, c->rowscale, c->Np, ncclUint64, ncclMax));  // non-negative doubles order as bits
      oz::k_rows_pow2<<<(unsigned)((c->Np + 255) / 256), 256, 0, c->stream>>>(c->N, c->Np, c->rowscale);
    }
    return 0;
  };
  if (src64) {
    CKR(row_scales(src64));
    oz::k_phi_colscale<double><<<(unsigned)((c->Dp + 255) / 256), 256, 0, c->stream>>>(src64, c->Dp, c->N, c->Dp,
                                                                                        c->rowscale, c->colscale);
    oz::k_phi_planes<double><<<16 * c->sm_count, 256, 0, c->stream>>>(src64, c->Dp, c->Np, c->Dp, c->rowscale,
                                                                      c->colscale, c->phiq, c->npa);
  } else {
    CKR(row_scales(c->phi));
    oz::k_phi_colscale<float><<<(unsigned)((c->Dp + 255) / 256), 256, 0, c->stream>>>(c->phi, c->Dp, c->N, c->Dp,
                                                                                       c->rowscale, c->colscale);
    oz::k_phi_planes<float><<<16 * c->sm_count, 256, 0, c->stream>>>(c->phi, c->Dp, c->Np, c->Dp, c->rowscale,
                                                                     c->colscale, c->phiq, c->npa);
  }
  c->launches += 3;
  if (c->phiqT) {
    const int64_t tiles = (c->Np / 64) * (c->Dp / 64);
    oz::k_planes_transpose<<<dim3((unsigned)std::min<int64_t>(tiles, 8 * c->sm_count), 1, c->npa), 256, 0, c->stream>>>(
        c->phiq, c->Np, c->Dp, c->phiqT);
    c->launches++;
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  c->oz_ready = true;
  return 0;
}

template <int QW>
int oz_init_kernels() {
  static DeviceFlags f_fwd, f_bwd, f_band, f_fwd3, f_bwd3;
  CKR(smem_attr_once(f_fwd, oz::contract_kernel<QW, oz::MODE_FWD>, oz::Cfg<QW>::SMEM));
  CKR(smem_attr_once(f_bwd, oz::contract_kernel<QW, oz::MODE_BWD>, oz::Cfg<QW>::SMEM));
  CKR(smem_attr_once(f_band, oz::contract_kernel<QW, oz::MODE_BAND>, oz::Cfg<QW>::SMEM));
  CKR(smem_attr_once(f_fwd3, oz::contract_kernel<QW, oz::MODE_FWD, 3>, oz::Cfg<QW, 3>::SMEM));
  CKR(smem_attr_once(f_bwd3, oz::contract_kernel<QW, oz::MODE_BWD, 3>, oz::Cfg<QW, 3>::SMEM));
  return 0;
}

// quantise columns [qoff, qoff+QW) of M (k_real rows, row stride ldm) into planes;
// colmax (QW entries) holds the column maxima when `colmax_ready`
template <typename T, int QW>
int oz_quantize(cofem_ctx* c, const T* M, int ldm, int qoff, int64_t k_real, int64_t k_pad, const double* pre,
                int8_t* planes, unsigned long long* colmax, bool colmax_ready, unsigned long long* reset,
                const Status* st, bool global_max = false) {
  if (!colmax_ready) {
    CK(cudaMemsetAsync(colmax, 0, QW * sizeof(unsigned long long), c->stream));
    const int bs = QW * (256 / QW);
    oz::k_colmax<T><<<2 * c->sm_count, bs, bs * sizeof(double), c->stream>>>(k_real, ldm, qoff, QW, M, pre, colmax,
                                                                             st);
    c->launches++;
  }
  // a time-sharded operand: every rank quantises with the global column
  // maxima, so halo rows received from a neighbour share this rank's scales
  if (global_max && c->nranks > 1) CKR(allreduce(c, colmax, QW, ncclUint64, ncclMax));
  const int64_t nchunk = k_pad / oz::QCHUNK_K;  // one warp each, 8 warps per block
  // one wave of resident blocks (3 / SM at <= 85 registers), grid-stride over the chunks
  oz::k_quantize<T, QW><<<(unsigned)std::min<int64_t>((nchunk + 7) / 8, 3 * c->sm_count), 256, 0, c->stream>>>(
      k_real, k_pad, ldm, qoff, M, pre, colmax, c->opscale, planes, reset, st);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// one persistent contraction launch; out = fp64 split partials [S][rows][QW]
template <int QW, bool BWD>
int oz_contract(cofem_ctx* c, const CUtensorMap& map_b, int64_t n_rows_out, int64_t k_total, const double* row_scale,
                double* out, int* nsplit_out, const Status* st) {
  CKR(oz_init_kernels<QW>());
  const int64_t n_mblocks = n_rows_out / oz::BM;
  const int64_t ntiles = k_total / oz::KT;
  SplitPlan sp = plan_splits(n_mblocks, ntiles, oz::KT, c->sm_count, (double)n_rows_out * QW * 8.0,
                             (double)c->Np * c->Dp * c->npa);
  // exact int32 accumulation: <= 4 digit products of <= 2^14 per significance
  // block, so keep K <= 2^15 per item
  while (sp.per_split > oz::MAX_K_PER_ITEM ||
         (size_t)sp.nsplit * n_rows_out * QW * 8 > (BWD ? c->ppart_cap : c->vpart_cap)) {
    if (sp.per_split > oz::MAX_K_PER_ITEM) sp.per_split = oz::MAX_K_PER_ITEM;
    else sp.per_split *= 2;
    sp.nsplit = (int)((k_total + sp.per_split - 1) / sp.per_split);
  }
  const int n_items = (int)(n_mblocks * sp.nsplit);
  const int grid = std::min(n_items, c->sm_count);
  // Phi^T V: the K-major transposed planes when present (same integers, same
  // splits -> bitwise the MN-major result, read like Phi P), else MN-major
  const bool trans = BWD && c->phiqT;
  const CUtensorMap& map_a = trans ? c->map_phiT : (BWD ? c->map_phi_bwd : c->map_phi_fwd);
  cudaEvent_t e0 = nullptr;
  if (c->time_kernels) {
    e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  auto go = [&](auto kern, size_t smem) {
    kern<<<grid, oz::NTHREADS, smem, c->stream>>>(map_a, map_b, (int)n_mblocks, n_items, sp.per_split, (int)k_total, 0,
                                                  row_scale, c->opscale, out, n_rows_out, n_rows_out, nullptr, st,
                                                  sp.nsplit, QW);
  };
  if (c->npa == 3) {
    if (BWD && !trans) go(oz::contract_kernel<QW, oz::MODE_BWD, 3>, oz::Cfg<QW, 3>::SMEM);
    else go(oz::contract_kernel<QW, oz::MODE_FWD, 3>, oz::Cfg<QW, 3>::SMEM);
  } else {
    if (BWD && !trans) go(oz::contract_kernel<QW, oz::MODE_BWD>, oz::Cfg<QW>::SMEM);
    else go(oz::contract_kernel<QW, oz::MODE_FWD>, oz::Cfg<QW>::SMEM);
  }
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({BWD ? 1 : 0, c->evnext - 2});
  }
  (void)e0;
  c->launches++;
  if (BWD) c->bwd_launches++;
  else c->fwd_launches++;
  CK(cudaGetLastError());
  *nsplit_out = sp.nsplit;
  return 0;
}

template <int QW>
int oz_fwd(cofem_ctx* c, const double* src, int lds, int qoff, double* vout, const Status* st) {
  CKR(ensure_oz(c));
  const int slot = QW / 8;
  if (!c->map_p_ok[slot]) {
    CKR(encode_u8_kblocked(&c->map_p[slot], c->pq, c->Dp, QW, QW));
    c->map_p_ok[slot] = true;
  }
  // P's column maxima come fused out of k_direction inside a PCG solve; the
  // quantiser resets the V maxima that k_sum_splits accumulates next
  CKR((oz_quantize<double, QW>(c, src, lds, qoff, c->D, c->Dp, c->colscale, c->pq, c->colmax + qoff,
                               c->p_colmax_valid, c->vcolmax, st, true)));  // shards: the unsharded P scales
  int ns = 1;
  CKR((oz_contract<QW, false>(c, c->map_p[slot], c->Np, c->Dp, c->rowscale, (double*)c->vpart, &ns, st)));
  const int bs = elem_block(QW);
  k_sum_splits<double><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
      c->Np, QW, ns, (const double*)c->vpart, vout, c->rowscale, c->vcolmax, st);
  c->launches++;
  CK(cudaGetLastError());
  c->v_colmax_valid = true;
  return 0;
}

template <int QW>
int oz_bwd(cofem_ctx* c, const double* v, int* nsplit_out, const Status* st) {
  CKR(ensure_oz(c));
  const int slot = QW / 8;
  if (!c->map_v_ok[slot]) {
    CKR(encode_u8_kblocked(&c->map_v[slot], c->vq, c->Np, QW, QW));
    c->map_v_ok[slot] = true;
  }
  CKR((oz_quantize<double, QW>(c, v, QW, 0, c->N, c->Np, c->rowscale, c->vq, c->vcolmax, c->v_colmax_valid,
                               nullptr, st)));
  c->v_colmax_valid = false;
  return oz_contract<QW, true>(c, c->map_v[slot], c->Dp, c->Np, c->colscale, (double*)c->ppart, nsplit_out, st);
}

// ---- banded Toeplitz (convolution) contractions ----------------------------
// (Phi p)_i = sum_m h_m p_{i-m}: every 128-row output tile multiplies the same
// lower band [4][128][128 + lpad] with the operand window starting lpad rows
// earlier; (Phi^T u)_j = sum_m h_m u_{j+m} uses the upper band and the window
// starting at the tile.  Ends of the sequence arrive as TMA zero fill.
// launch the band contraction: smem-resident band when it fits, else the
// streaming MODE_BAND of contract_kernel
template <int QW, int NPA>
int launch_band_t(cofem_ctx* c, const CUtensorMap& map_a, const CUtensorMap& map_b, int nmb, int nk, int offset,
                  double* out, int64_t out_rows, int64_t rows_real, unsigned long long* colmax, const Status* st) {
  const int grid = std::min(nmb, c->sm_count);
  const size_t sm = oz::BandCfg<QW, NPA>::smem(nk);
  if (sm <= 227 * 1024) {
    static DeviceFlags flags;
    CKR(smem_attr_once(flags, oz::band_kernel<QW, oz::EPI_PLAIN, NPA>, 227 * 1024));
    oz::band_kernel<QW, oz::EPI_PLAIN, NPA><<<grid, oz::BAND_NTHREADS, sm, c->stream>>>(
        map_a, map_b, nmb, nk, offset, c->hrows, c->opscale, out, rows_real, colmax, st, oz::BandStep{});
  } else {
    static DeviceFlags flags;
    CKR(smem_attr_once(flags, oz::contract_kernel<QW, oz::MODE_BAND, NPA>, oz::Cfg<QW, NPA>::SMEM));
    oz::contract_kernel<QW, oz::MODE_BAND, NPA><<<grid, oz::NTHREADS, oz::Cfg<QW, NPA>::SMEM, c->stream>>>(
        map_a, map_b, nmb, nmb, nk, 0, offset, c->hrows, c->opscale, out, out_rows, rows_real, colmax, st);
  }
  CK(cudaGetLastError());
  return 0;
}
template <int QW>
int launch_band(cofem_ctx* c, const CUtensorMap& map_a, const CUtensorMap& map_b, int nmb, int nk, int offset,
                double* out, int64_t out_rows, int64_t rows_real, unsigned long long* colmax, const Status* st) {
  if (c->npa == 3) return launch_band_t<QW, 3>(c, map_a, map_b, nmb, nk, offset, out, out_rows, rows_real, colmax, st);
  return launch_band_t<QW, 4>(c, map_a, map_b, nmb, nk, offset, out, out_rows, rows_real, colmax, st);
}

// V -> operand planes for Phi^T (global column maxima), then the halo: the
// right neighbour's first lpad rows land after this shard's Np rows
template <int QW>
int conv_quantize_v(cofem_ctx* c, const double* v, const Status* st) {
  const int slot = QW / 8;
  const int64_t lp = c->conv_lpad;
  const bool right = c->nranks > 1 && c->rank < c->nranks - 1;
  if (!c->map_v_ok[slot]) {
    CKR(encode_u8_kblocked(&c->map_v[slot], c->vq, c->Np + (right ? lp : 0), QW, QW));
    c->map_v_ok[slot] = true;
  }
  CKR((oz_quantize<double, QW>(c, v, QW, 0, c->N, c->Np, nullptr, c->vq, c->vcolmax, c->v_colmax_valid,
                               nullptr, st, true)));  // band operands carry no scale (hrows holds it)
  c->v_colmax_valid = false;
  return halo_exchange(c, c->vq, c->vq + c->Np * 4 * QW, (size_t)lp * 4 * QW, -1);
}

template <int QW>
int conv_fwd(cofem_ctx* c, const double* src, int lds, int qoff, double* vout, const Status* st) {
  CKR(oz_init_kernels<QW>());
  const int slot = QW / 8;
  const int64_t lp = c->conv_lpad;
  const bool left = c->nranks > 1 && c->rank > 0;  // a left neighbour's rows precede the data
  if (!c->map_p_ok[slot]) {
    if (left) CKR(encode_u8_kblocked(&c->map_p[slot], c->pq - lp * 4 * QW, lp + c->Dp, QW, QW));
    else CKR(encode_u8_kblocked(&c->map_p[slot], c->pq, c->Dp, QW, QW));
    c->map_p_ok[slot] = true;
  }
  CKR((oz_quantize<double, QW>(c, src, lds, qoff, c->D, c->Dp, nullptr, c->pq, c->colmax + qoff,
                               c->p_colmax_valid, c->vcolmax, st, true)));
  // halo: this shard's last lpad operand rows become the right neighbour's
  // first window rows (K-blocked planes: lpad / 64 contiguous blocks)
  CKR(halo_exchange(c, c->pq + std::max<int64_t>(c->D - lp, 0) * 4 * QW, c->pq - lp * 4 * QW,
                    (size_t)lp * 4 * QW, +1));
  const int nmb = (int)(c->Np / oz::BM);
  if (c->time_kernels) {
    cudaEvent_t e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  CKR(launch_band<QW>(c, c->map_band_fwd, c->map_p[slot], nmb, oz::BM + c->conv_lpad, left ? 0 : -c->conv_lpad,
                      vout, c->Np, c->N, c->vcolmax, st));
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({0, c->evnext - 2});
  }
  c->launches++;
  c->fwd_launches++;
  CK(cudaGetLastError());
  c->v_colmax_valid = true;
  return 0;
}

template <int QW>
int conv_bwd(cofem_ctx* c, const double* v, int* nsplit_out, const Status* st) {
  CKR(oz_init_kernels<QW>());
  CKR(conv_quantize_v<QW>(c, v, st));
  const int nmb = (int)(c->Dp / oz::BM);
  if (c->time_kernels) {
    cudaEvent_t e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  CKR(launch_band<QW>(c, c->map_band_adj, c->map_v[QW / 8], nmb, oz::BM + c->conv_lpad, 0, (double*)c->ppart,
                      c->Dp, c->D, nullptr, st));
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({1, c->evnext - 2});
  }
  c->launches++;
  c->bwd_launches++;
  CK(cudaGetLastError());
  *nsplit_out = 1;
  return 0;
}

// Phi^T V of a PCG step with the combine fused into the band epilogue:
// Psi[:, qoff:qoff+QW] = beta Phi^T V + alpha .* P and pi[qoff:...] directly
// (no U round trip, no k_combine).  Returns 1 when the band does not fit the
// smem-resident kernel (caller falls back to conv_bwd + k_combine).
template <int QW, int NPA>
int conv_bwd_comb_t(cofem_ctx* c, const double* v, int qoff, double beta, const Status* st) {
  const int nk = oz::BM + c->conv_lpad;
  const size_t sm = oz::BandCfg<QW, NPA>::smem(nk);
  if (sm > 227 * 1024 - 64) return 1;  // (the last-block fold adds a little static smem)
  CKR(oz_init_kernels<QW>());
  CKR(conv_quantize_v<QW>(c, v, st));
  const int nmb = (int)(c->Dp / oz::BM);
  const int grid = std::min(nmb, std::min(c->sm_count, c->nblk_elem));
  static DeviceFlags flags;
  CKR(smem_attr_once(flags, oz::band_kernel<QW, oz::EPI_COMB, NPA>, 227 * 1024 - 64));
  if (c->time_kernels) {
    cudaEvent_t e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  Scalars sc = c->sc();
  CK(cudaGetLastError());
  oz::BandStep bs{};
  bs.P = (const double*)c->P + qoff;
  bs.ld = c->ldq;
  bs.alpha = c->alpha;
  bs.beta = beta;
  bs.out0 = sc.pi + qoff;
  bs.partials = sc.partials;
  bs.ticket = sc.ticket + 1;
  oz::band_kernel<QW, oz::EPI_COMB, NPA><<<grid, oz::BAND_NTHREADS, sm, c->stream>>>(
      c->map_band_adj, c->map_v[QW / 8], nmb, nk, 0, c->hrows, c->opscale, (double*)c->Psi + qoff, c->D, nullptr, st,
      bs);
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({1, c->evnext - 2});
  }
  c->launches++;
  c->bwd_launches++;
  CK(cudaGetLastError());
  return 0;
}

template <int QW>
int conv_bwd_comb(cofem_ctx* c, const double* v, int qoff, double beta, const Status* st) {
  return c->npa == 3 ? conv_bwd_comb_t<QW, 3>(c, v, qoff, beta, st) : conv_bwd_comb_t<QW, 4>(c, v, qoff, beta, st);
}

// ---- convolution, float64 FFT path (dct.cuh k_conv_fft_pass) ----------------
// dst (D x ldq) = Phi src (adj: Phi^T src) for all ldq columns at once
int conv_fft_pass(cofem_ctx* c, const double* src, double* dst, bool adj, const Status* stt) {
  constexpr int N1 = 32, N2 = 32, FPI = DCT_FPI, NT = FPI * N2;
  constexpr size_t smem = (size_t)FPI * dctf::region_entries(N1, N2) * sizeof(double2);
  static DeviceFlags flags;
  CKR(smem_attr_once(flags, dctf::k_conv_fft_pass<N1, N2>, smem));
  const int L = c->conv_L, valid = CONV_FFT_N - (L - 1);
  const int nblocks = (int)((c->D + valid - 1) / valid);
  const int items = nblocks * (c->ldq / (2 * FPI));
  const int per_sm = std::min(16, std::max(1, (int)((228 * 1024) / (smem + 1024))));
  const int grid = std::min(items, per_sm * c->sm_count);
  dctf::k_conv_fft_pass<N1, N2><<<grid, NT, smem, c->stream>>>(src, dst, c->D, c->ldq, c->ldq / (2 * FPI), nblocks, valid,
                                                                adj ? 0 : L - 1, L - 1, adj ? c->cf_Hr : c->cf_H,
                                                                c->dct_wN, stt);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// Psi = beta Phi^T Phi P + alpha .* P, pi: two FFT passes + the streaming combine
int conv_fft_system_apply(cofem_ctx* c, double beta, const Status* stt) {
  cudaEvent_t e0 = nullptr;
  if (c->time_kernels) {
    e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  CKR(conv_fft_pass(c, (const double*)c->P, (double*)c->V, false, stt));
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({0, c->evnext - 2});
    c->fwd_launches++;
  }
  (void)e0;
  CKR(conv_fft_pass(c, (const double*)c->V, (double*)c->tmpD, true, stt));
  Scalars sc = c->sc();
  const int bs = elem_block(c->ldq);
  k_combine<double><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
      c->Dp, c->ldq, 0, c->ldq, 1, (const double*)c->tmpD, beta, c->alpha, (const double*)c->P, (double*)c->Psi, sc,
      stt);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// ---- 2-D partial DCT: fused float64 FFT passes (dct.cuh) ------------------
// pass over an n x n x ldq block; row passes run along j (outer i), column
// passes along i (outer j / l)
template <int N1, int N2, int MODE, bool VV = false>
int dct_pass_t(cofem_ctx* c, const double* src, double* dst, bool rows, const Status* stt,
               const dctf::VvArgs& vv = dctf::VvArgs()) {
  const int64_t n = c->dct_n, ldq = c->ldq;
  constexpr int FPI = DCT_FPI, NT = FPI * N2;
  constexpr size_t smem = (size_t)FPI * dctf::region_entries(N1, N2) * sizeof(double2) + N1 * N2;  // FFT regions + mask column
  static_assert(!VV || (size_t)N1 * N2 >= ((NT + 31) / 32) * dctf::VV_MAXQ * sizeof(double), "vv accumulators reuse the mask column");
  static DeviceFlags flags;
  CKR(smem_attr_once(flags, dctf::k_dct_pass<N1, N2, MODE, FPI, VV>, smem));
  const int items = (int)(n * (ldq / (2 * FPI)));
  int per_sm = std::max(1, (int)((228 * 1024) / (smem + 1024)));  // blocks that fit one SM's shared memory
  if (per_sm > 16) per_sm = 16;
  const int grid = std::min(items, per_sm * c->sm_count);
  if (VV) c->dct_vv_blocks = grid;
  dctf::k_dct_pass<N1, N2, MODE, FPI, VV><<<grid, NT, smem, c->stream>>>(
      src, dst, rows ? n * ldq : ldq, rows ? ldq : n * ldq, (int)n, (int)(ldq / (2 * FPI)), c->dct_wN, c->dct_tw,
      c->dct_gridT, stt, c->dct_wT, vv);
  c->launches++;
  return 0;
}

// n = 1024: one warp per complex FFT, data in registers (dct1024.cuh)
template <int MODE>
int dct_pass_w(cofem_ctx* c, const double* src, double* dst, bool rows, const Status* stt) {
  const int64_t n = c->dct_n, ldq = c->ldq;
  static DeviceFlags flags;
  CKR(smem_attr_once(flags, dctw::k_pass<MODE>, dctw::SMEM));
  const int items = (int)(n * (ldq / 2));
  const int grid = std::min((items + dctw::WARPS - 1) / dctw::WARPS, c->sm_count);
  dctw::k_pass<MODE><<<grid, 32 * dctw::WARPS, dctw::SMEM, c->stream>>>(
      src, dst, (int)((rows ? n * ldq : ldq) / 2), (int)((rows ? ldq : n * ldq) / 2), (int)n, (int)(ldq / 2), c->dct_twF,
      c->dct_tw, c->dct_pm, stt);
  c->launches++;
  return 0;
}

template <int MODE>
int dct_pass(cofem_ctx* c, const double* src, double* dst, bool rows, const Status* stt) {
  if (c->dct_n == 1024 && c->dct_pm) {
    CKR((dct_pass_w<MODE>(c, src, dst, rows, stt)));
    CK(cudaGetLastError());
    return 0;
  }
  switch (c->dct_n) {
    case 64: CKR((dct_pass_t<8, 8, MODE>(c, src, dst, rows, stt))); break;
    case 128: CKR((dct_pass_t<8, 16, MODE>(c, src, dst, rows, stt))); break;
    case 256: CKR((dct_pass_t<16, 16, MODE>(c, src, dst, rows, stt))); break;
    case 512: CKR((dct_pass_t<16, 32, MODE>(c, src, dst, rows, stt))); break;
    case 1024: CKR((dct_pass_t<32, 32, MODE>(c, src, dst, rows, stt))); break;
    default: return fail(COFEM_EINVAL, "unsupported DCT image side");
  }
  CK(cudaGetLastError());
  return 0;
}

// bufB <- coefficient grid Y[(k n + l) ldq + q] = DCT2 of every column image of P
int dct_forward_dev(cofem_ctx* c, const double* P, const Status* stt) {
  CKR((dct_pass<dctf::P_FWD>(c, P, c->bufA, true, stt)));
  return dct_pass<dctf::P_FWD>(c, c->bufA, c->bufB, false, stt);
}

// out <- DCT2^T of the coefficient grid in bufB
int dct_adjoint_dev(cofem_ctx* c, double* out, const Status* stt) {
  CKR((dct_pass<dctf::P_INV>(c, c->bufB, c->bufA, false, stt)));
  return dct_pass<dctf::P_INV>(c, c->bufA, out, true, stt);
}

// Psi = beta Phi^T Phi P + alpha .* P for all ldq columns at once, pi on the
// fly: row DCT-II, fused column DCT-II / mask / DCT-III, row DCT-III + combine
int dct_system_apply(cofem_ctx* c, double beta, const Status* stt) {
  tick(c, -1);
  CKR((dct_pass<dctf::P_FWD>(c, (const double*)c->P, c->bufA, true, stt)));
  tick(c, 0);
  cudaEvent_t e0 = nullptr;
  if (c->time_kernels) {
    e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  CKR((dct_pass<dctf::P_FMI>(c, c->bufA, c->bufB, false, stt)));
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({0, c->evnext - 2});
    c->fwd_launches++;
  }
  (void)e0;
  tick(c, 1);
  // the row DCT-III writes Z; Psi = beta Z + alpha .* P and pi in the streaming
  // combine (fusing it into the pass stalls the FFT pipeline on the P loads)
  CKR((dct_pass<dctf::P_INV>(c, c->bufB, c->bufA, true, stt)));
  tick(c, 2);
  Scalars sc = c->sc();
  const int bs = elem_block(c->ldq);
  k_combine<double><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
      c->Dp, c->ldq, 0, c->ldq, 1, (const double*)c->bufA, beta, c->alpha, (const double*)c->P, (double*)c->Psi, sc,
      stt);
  c->launches++;
  tick(c, 3);
  CK(cudaGetLastError());
  return 0;
}

// The Psi-free PCG step of a 2-D DCT system (one GPU, K + 1 <= 32, n >= 512): the three
// passes with vv = ||Z||^2 out of the last one, then k_update_psi (pcg.cuh) instead of
// k_combine + k_update.  bufA <- Z = Phi^T Phi P.  0.4 GB less per step.  (A first version
// took <P, alpha P> from a direction kernel with one more reduction: that kernel ran 77 us
// slower live than under ncu -- COFEM_TICKS, profiles/r2aj_* -- and the step lost 1.4 %; now
// the term follows the direction recurrence from two inner products of k_update_psi.)
bool dct_psifree_eligible(const cofem_ctx* c) {
  return c->kind == 2 && c->nranks <= 1 && c->ldq <= dctf::VV_MAXQ && c->dct_n >= 512 && !c->dct_pm && c->dct_fscal &&
         !getenv("COFEM_DCT_PSI");
}

int dct_apply_vv(cofem_ctx* c, const Status* stt) {
  tick(c, -1);
  CKR((dct_pass<dctf::P_FWD>(c, (const double*)c->P, c->bufA, true, stt)));
  tick(c, 0);
  if (c->time_kernels) cudaEventRecord(next_event(c), c->stream);
  CKR((dct_pass<dctf::P_FMI>(c, c->bufA, c->bufB, false, stt)));
  if (c->time_kernels) {
    cudaEventRecord(next_event(c), c->stream);
    c->timed.push_back({0, c->evnext - 2});
    c->fwd_launches++;
  }
  tick(c, 1);
  dctf::VvArgs vv;
  vv.partials = c->dct_partials;
  vv.ldq = c->ldq;
  if (c->dct_n == 1024) CKR((dct_pass_t<32, 32, dctf::P_INV, true>(c, c->bufB, c->bufA, true, stt, vv)));
  else CKR((dct_pass_t<16, 32, dctf::P_INV, true>(c, c->bufB, c->bufA, true, stt, vv)));
  tick(c, 2);
  CK(cudaGetLastError());
  return 0;
}

// ---- 1-D subsampled DCT (kind 3; dct1.cuh) ----------------------------------
int dct1_plan(cofem_ctx* c) {
  const int hc = c->ldq / 2;
  if (c->fft_plan_hc == hc) return 0;
  CKR(cufft_load());
  if (c->fft_plan_hc) g_cufft.destroy(c->fft_plan);
  c->fft_plan_hc = 0;
  int n = (int)c->D, emb = (int)c->D;
  if (g_cufft.planMany(&c->fft_plan, 1, &n, &emb, hc, 1, &emb, hc, 1, CUFFT_Z2Z, hc) != CUFFT_SUCCESS)
    return fail(COFEM_ECUDA, "cufftPlanMany failed");
  if (g_cufft.setStream(c->fft_plan, c->stream) != CUFFT_SUCCESS) return fail(COFEM_ECUDA, "cufftSetStream failed");
  c->fft_plan_hc = hc;
  return 0;
}

int dct1_fft(cofem_ctx* c, int dir) {
  CKR(dct1_plan(c));
  cufftDoubleComplex* z = reinterpret_cast<cufftDoubleComplex*>(c->bufA);
  if (g_cufft.execZ2Z(c->fft_plan, z, z, dir) != CUFFT_SUCCESS) return fail(COFEM_ECUDA, "cufftExecZ2Z failed");
  c->launches++;
  return 0;
}

// bufA <- DCT-III of the real block X (all ldq columns), in v order
int dct1_inverse(cofem_ctx* c, const double* X) {
  dct1::k_pre<<<8 * c->sm_count, 256, 0, c->stream>>>(c->D, c->ldq, X, reinterpret_cast<double2*>(c->bufA));
  c->launches++;
  CK(cudaGetLastError());
  return dct1_fft(c, CUFFT_INVERSE);
}

// out (real [Dp][ldq]) <- orthonormal DCT-II of the v-order vectors in bufA
int dct1_forward_post(cofem_ctx* c, double* out) {
  CKR(dct1_fft(c, CUFFT_FORWARD));
  dct1::k_post<<<8 * c->sm_count, 256, 0, c->stream>>>(c->D, c->Dp, c->ldq, reinterpret_cast<const double2*>(c->bufA),
                                                       out);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// Psi = beta Phi^T Phi P + alpha .* P for all ldq columns, pi on the fly:
// DCT-III, mask (v order), DCT-II, then the streaming PCG combine
int dct1_system_apply(cofem_ctx* c, double beta, const Status* stt) {
  CKR(dct1_inverse(c, (const double*)c->P));
  dct1::k_vmask<<<8 * c->sm_count, 256, 0, c->stream>>>(c->D, c->ldq / 2, reinterpret_cast<double2*>(c->bufA),
                                                        c->dct1_mv);
  c->launches++;
  CK(cudaGetLastError());
  CKR(dct1_forward_post(c, (double*)c->tmpD));
  Scalars sc = c->sc();
  const int bs = elem_block(c->ldq);
  k_combine<double><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
      c->Dp, c->ldq, 0, c->ldq, 1, (const double*)c->tmpD, beta, c->alpha, (const double*)c->P, (double*)c->Psi, sc,
      stt);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// tmpD <- Phi^T of the N x ldq block in V
int dct1_adjoint_from_V(cofem_ctx* c) {
  CK(cudaMemsetAsync(c->bufA, 0, (size_t)c->D * c->ldq * sizeof(double), c->stream));
  dct1::k_scatter<<<8 * c->sm_count, 256, 0, c->stream>>>(c->N, c->D, c->ldq, c->dct_mask, (const double*)c->V,
                                                          reinterpret_cast<double2*>(c->bufA));
  c->launches++;
  CK(cudaGetLastError());
  return dct1_forward_post(c, (double*)c->tmpD);
}

// ---- the two contractions ----------------------------------------------
// fwd: V (Np x qpc dense) = Phi * src[:, qoff:qoff+qpc]  (src Dp x lds)
template <typename T, int QP, typename PhiT>
int run_fwd_cc(cofem_ctx* c, const PhiT* phi, const T* src, int lds, int qoff, T* vout, const Status* st);
template <typename T, int QP, typename PhiT>
int run_bwd_cc(cofem_ctx* c, const PhiT* phi, const T* v, int* nsplit_out, const Status* st);

template <typename T, int QP>
int run_fwd(cofem_ctx* c, const T* src, int lds, int qoff, T* vout, const Status* st) {
  if constexpr (std::is_same<T, double>::value) {
    if (c->kind == 1) return conv_fwd<QP>(c, src, lds, qoff, vout, st);
    if (c->prec == COFEM_OZAKI) return oz_fwd<QP>(c, src, lds, qoff, vout, st);
  }
  if constexpr (std::is_same<T, double>::value) {
    if (c->phi64) return run_fwd_cc<T, QP, double>(c, c->phi64, src, lds, qoff, vout, st);
  }
  return run_fwd_cc<T, QP, float>(c, c->phi, src, lds, qoff, vout, st);
}

// the CUDA-core contraction over a float32 or float64 dictionary
template <typename T, int QP, typename PhiT>
int run_fwd_cc(cofem_ctx* c, const PhiT* phi, const T* src, int lds, int qoff, T* vout, const Status* st) {
  using K = Kern<T, QP, PhiT>;
  CKR(K::init());
  const int64_t ntiles = c->Dp / Tiles<T>::FBK;
  const int64_t mblocks = c->Np / K::FC::BM;
  SplitPlan sp = plan_splits(mblocks, ntiles, Tiles<T>::FBK, K::fwd_occ * c->sm_count,
                             (double)c->Np * QP * sizeof(T), (double)c->Np * c->Dp * 4.0);
  while ((size_t)sp.nsplit * c->Np * QP * sizeof(T) > c->vpart_cap) {  // capacity guard
    sp.per_split *= 2;
    sp.nsplit = (int)((c->Dp + sp.per_split - 1) / sp.per_split);
  }
  dim3 grid((unsigned)mblocks, (unsigned)sp.nsplit);
  if (c->time_kernels) {
    cudaEvent_t e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  K::fwd<<<grid, K::FC::NT, K::FC::SMEM, c->stream>>>(phi, c->Dp, src, lds, qoff, sp.per_split, c->Dp,
                                                      (T*)c->vpart, c->Np, st);
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({0, c->evnext - 2});
  }
  c->launches++;
  c->fwd_launches++;
  CK(cudaGetLastError());
  const int bs = elem_block(QP);
  k_sum_splits<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(c->Np, QP, sp.nsplit, (const T*)c->vpart,
                                                                        vout, nullptr, nullptr, st);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// bwd: ppart = Phi^T V  (V Np x QP dense); returns number of splits
template <typename T, int QP>
int run_bwd(cofem_ctx* c, const T* v, int* nsplit_out, const Status* st) {
  if constexpr (std::is_same<T, double>::value) {
    if (c->kind == 1) return conv_bwd<QP>(c, v, nsplit_out, st);
    if (c->prec == COFEM_OZAKI) return oz_bwd<QP>(c, v, nsplit_out, st);
  }
  if constexpr (std::is_same<T, double>::value) {
    if (c->phi64) return run_bwd_cc<T, QP, double>(c, c->phi64, v, nsplit_out, st);
  }
  return run_bwd_cc<T, QP, float>(c, c->phi, v, nsplit_out, st);
}

template <typename T, int QP, typename PhiT>
int run_bwd_cc(cofem_ctx* c, const PhiT* phi, const T* v, int* nsplit_out, const Status* st) {
  using K = Kern<T, QP, PhiT>;
  CKR(K::init());
  const int64_t ntiles = c->Np / Tiles<T>::BBK;
  const int64_t nblocks = c->Dp / K::BC::BN;
  SplitPlan sp = plan_splits(nblocks, ntiles, Tiles<T>::BBK, K::bwd_occ * c->sm_count,
                             (double)c->Dp * QP * sizeof(T), (double)c->Np * c->Dp * 4.0);
  while ((size_t)sp.nsplit * c->Dp * QP * sizeof(T) > c->ppart_cap) {
    sp.per_split *= 2;
    sp.nsplit = (int)((c->Np + sp.per_split - 1) / sp.per_split);
  }
  dim3 grid((unsigned)nblocks, (unsigned)sp.nsplit);
  if (c->time_kernels) {
    cudaEvent_t e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  K::bwd<<<grid, K::BC::NT, K::BC::SMEM, c->stream>>>(phi, c->Dp, v, QP, 0, sp.per_split, c->Np,
                                                      (T*)c->ppart, c->Dp, st);
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({1, c->evnext - 2});
  }
  c->launches++;
  c->bwd_launches++;
  CK(cudaGetLastError());
  *nsplit_out = sp.nsplit;
  return 0;
}

template <typename T>
int fwd_chunk(cofem_ctx* c, int qpc, const T* src, int lds, int qoff, T* vout, const Status* st) {
  switch (qpc) {
    case 8: return run_fwd<T, 8>(c, src, lds, qoff, vout, st);
    case 16: return run_fwd<T, 16>(c, src, lds, qoff, vout, st);
    case 24: return run_fwd<T, 24>(c, src, lds, qoff, vout, st);
    case 32: return run_fwd<T, 32>(c, src, lds, qoff, vout, st);
  }
  return fail(COFEM_EINVAL, "bad column chunk");
}

template <typename T>
int bwd_chunk(cofem_ctx* c, int qpc, const T* v, int* ns, const Status* st) {
  switch (qpc) {
    case 8: return run_bwd<T, 8>(c, v, ns, st);
    case 16: return run_bwd<T, 16>(c, v, ns, st);
    case 24: return run_bwd<T, 24>(c, v, ns, st);
    case 32: return run_bwd<T, 32>(c, v, ns, st);
  }
  return fail(COFEM_EINVAL, "bad column chunk");
}

inline int chunk_width(int ldq, int qoff) { return std::min(QCHUNK, ldq - qoff); }

// Psi = beta Phi^T Phi P + alpha .* P for all ldq columns, pi on the fly
template <typename T>
int system_apply_dev(cofem_ctx* c, double beta, const Status* st) {
  if constexpr (std::is_same<T, double>::value) {
    if (c->kind == 2) return dct_system_apply(c, beta, st);
    if (c->kind == 3) return dct1_system_apply(c, beta, st);
    if (c->conv_fft) return conv_fft_system_apply(c, beta, st);
  }
  Scalars sc = c->sc();
  for (int qoff = 0; qoff < c->ldq; qoff += QCHUNK) {
    const int qpc = chunk_width(c->ldq, qoff);
    CKR(fwd_chunk<T>(c, qpc, (const T*)c->P, c->ldq, qoff, (T*)c->V, st));
    CKR(reduce_partial_v(c, (size_t)c->Np * qpc, nccl_t<T>()));
    if constexpr (std::is_same<T, double>::value) {
      if (c->kind == 1) {  // convolution: combine fused into the band epilogue
        int rc = 1;
        switch (qpc) {
          case 8: rc = conv_bwd_comb<8>(c, (const double*)c->V, qoff, beta, st); break;
          case 16: rc = conv_bwd_comb<16>(c, (const double*)c->V, qoff, beta, st); break;
          case 24: rc = conv_bwd_comb<24>(c, (const double*)c->V, qoff, beta, st); break;
          case 32: rc = conv_bwd_comb<32>(c, (const double*)c->V, qoff, beta, st); break;
        }
        if (rc < 0) return rc;
        if (rc == 0) continue;
      }
    }
    int ns = 1;
    CKR(bwd_chunk<T>(c, qpc, (const T*)c->V, &ns, st));
    const int bs = elem_block(qpc);
    k_combine<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
        c->Dp, c->ldq, qoff, qpc, ns, (const T*)c->ppart, beta, c->alpha, (const T*)c->P, (T*)c->Psi, sc, st);
    c->launches++;
    CK(cudaGetLastError());
  }
  return 0;
}

// ---- fused convolution PCG step ---------------------------------------------
// One GPU, one column chunk (K + 1 <= 32), one preconditioner group, the
// smem-resident band: per PCG step four launches instead of six and no Psi
// block:
//   K1 band Phi P (EPI_FWD): V, column maxima of |V|, vv = ||V||^2
//   K2 k_quantize(V) (the exact maxima from K1; zeroes the |M^-1 R| maxima)
//   K3 band Phi^T V (EPI_UPD): gamma = rho / (beta vv + pap), R -= gamma Psi
//      on the fly, rho_new, ||R||^2, maxima of |M^-1 R|
//   K4 k_direction_q: stopping test, X, P(u+1) and its digit planes against
//      the bound scale, maxima of |P(u+1)|, pap = <P(u+1), alpha P(u+1)>
bool conv_fused_eligible(cofem_ctx* c, int ngroups) {
  if (!(c->kind == 1 && c->prec == COFEM_OZAKI && !c->conv_fft && c->nranks <= 1 && c->ldq <= QCHUNK &&
        ngroups == 1 && !c->conv_fused_off && c->fz_max))
    return false;
  const int nk = oz::BM + c->conv_lpad;
  return oz::BandCfg<32, 4>::smem(nk) <= 227 * 1024 - 64 - 512;
}

template <int QW, int NPA>
int conv_fused_launch(cofem_ctx* c, int which, int step, double beta, int q_real, const cofem_cg_config* cg,
                      Status* mirror) {
  const int slot = QW / 8;
  const int nk = oz::BM + c->conv_lpad;
  const int nmb = (int)(c->Np / oz::BM);
  const size_t sm = oz::BandCfg<QW, NPA>::smem(nk);
  const int ldq = c->ldq;
  Scalars sc = c->sc();
  double* vv = c->scal + 8 * ldq;
  double* pap = c->scal + 9 * ldq;
  unsigned long long* pmax[2] = {c->fz_max, c->fz_max + 32};
  unsigned long long* wmax = c->fz_max + 64;
  if (which == 0 || which == 2) {  // the band launches
    static DeviceFlags f1, f3;
    CKR(smem_attr_once(f1, oz::band_kernel<QW, oz::EPI_FWD, NPA>, 227 * 1024 - 64));
    CKR(smem_attr_once(f3, oz::band_kernel<QW, oz::EPI_UPD, NPA>, 227 * 1024 - 64));
    const int grid = std::min(nmb, std::min(c->sm_count, c->nblk_elem));
    oz::BandStep bs{};
    bs.ld = ldq;
    bs.q_real = q_real;
    bs.printed = cg->printed_recursion;
    bs.alpha = c->alpha;
    bs.minv = c->minv;
    bs.ngroups = 1;
    bs.beta = beta;
    bs.partials = sc.partials;
    cudaEvent_t e0 = nullptr;
    if (c->time_kernels) {
      e0 = next_event(c);
      cudaEventRecord(e0, c->stream);
    }
    if (which == 0) {
      if (!c->map_p_ok[slot]) {
        CKR(encode_u8_kblocked(&c->map_p[slot], c->pq, c->Dp, QW, QW));
        c->map_p_ok[slot] = true;
      }
      bs.out0 = vv;
      bs.ticket = sc.ticket + 3;
      oz::band_kernel<QW, oz::EPI_FWD, NPA><<<grid, oz::BAND_NTHREADS, sm, c->stream>>>(
          c->map_band_fwd, c->map_p[slot], nmb, nk, -c->conv_lpad, c->hrows, c->opscale, (double*)c->V, c->N,
          c->vcolmax, c->st, bs);
      c->fwd_launches++;
    } else {
      if (!c->map_v_ok[slot]) {
        CKR(encode_u8_kblocked(&c->map_v[slot], c->vq, c->Np, QW, QW));
        c->map_v_ok[slot] = true;
      }
      bs.P = (const double*)c->P;
      bs.R = (double*)c->R;
      bs.rho = sc.rho[step & 1];
      bs.vv = vv;
      bs.pap = pap;
      bs.gam_out = sc.gam[step & 1];
      bs.frozen = sc.frozen;
      bs.wmax = wmax;
      bs.reset = pmax[(step + 1) & 1];
      bs.out0 = sc.rho_new;
      bs.out1 = sc.rn2;
      bs.ticket = sc.ticket + 4;
      oz::band_kernel<QW, oz::EPI_UPD, NPA><<<grid, oz::BAND_NTHREADS, sm, c->stream>>>(
          c->map_band_adj, c->map_v[slot], nmb, nk, 0, c->hrows, c->opscale, nullptr, c->D, nullptr, c->st, bs);
      c->bwd_launches++;
    }
    if (c->time_kernels) {
      cudaEvent_t e1 = next_event(c);
      cudaEventRecord(e1, c->stream);
      c->timed.push_back({which == 0 ? 0 : 1, c->evnext - 2});
    }
    (void)e0;
  } else if (which == 1) {  // K2
    CKR((oz_quantize<double, QW>(c, (const double*)c->V, QW, 0, c->N, c->Np, nullptr, c->vq, c->vcolmax, true, wmax,
                                 c->st)));
    return 0;
  } else {  // K4 (step 0: the first direction; P in place, no X)
    const int64_t ngrp = c->Dp / 128;
    const unsigned grid = (unsigned)std::min<int64_t>(ngrp, 2 * c->sm_count);  // 2 blocks / SM resident
    const bool first = step == 0;
    oz::k_direction_q<QW><<<grid, 256, 0, c->stream>>>(
        c->Dp, q_real, step, cg->max_steps, cg->tolerance, cg->printed_recursion, (double*)c->P, (const double*)c->R,
        c->minv, c->alpha, sc, pmax[step & 1], pmax[(step + 1) & 1], wmax, c->vcolmax, c->opscale, c->pq, pap,
        sc.ticket + 5, c->st, mirror, first ? nullptr : (double*)c->X, first ? nullptr : (double*)c->P2,
        first ? nullptr : (const double*)c->P2);
  }
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

int conv_fused(cofem_ctx* c, int which, int step, double beta, int q_real, const cofem_cg_config* cg,
               Status* mirror = nullptr) {
  const bool p3 = c->npa == 3;
  switch (c->ldq) {
    case 8: return p3 ? conv_fused_launch<8, 3>(c, which, step, beta, q_real, cg, mirror)
                      : conv_fused_launch<8, 4>(c, which, step, beta, q_real, cg, mirror);
    case 16: return p3 ? conv_fused_launch<16, 3>(c, which, step, beta, q_real, cg, mirror)
                       : conv_fused_launch<16, 4>(c, which, step, beta, q_real, cg, mirror);
    case 24: return p3 ? conv_fused_launch<24, 3>(c, which, step, beta, q_real, cg, mirror)
                       : conv_fused_launch<24, 4>(c, which, step, beta, q_real, cg, mirror);
    case 32: return p3 ? conv_fused_launch<32, 3>(c, which, step, beta, q_real, cg, mirror)
                       : conv_fused_launch<32, 4>(c, which, step, beta, q_real, cg, mirror);
  }
  return fail(COFEM_EINVAL, "fused convolution step: unsupported column count");
}

// ---- one-launch PCG solve (persistent.cuh) --------------------------------
// dense dictionary, int8 path, one GPU, one column chunk, one preconditioner group
bool persistent_eligible(cofem_ctx* c, int ngroups) {
  return c->kind == 0 && c->prec == COFEM_OZAKI && c->nranks <= 1 && c->phiqT && c->ldq <= QCHUNK &&
         ngroups == 1 && !c->persistent_off;
}

// split plan of one contraction phase (the constraints of oz_contract)
SplitPlan persistent_splits(cofem_ctx* c, int64_t rows_out, int64_t k_total, size_t cap, int QW) {
  SplitPlan sp = plan_splits(rows_out / oz::BM, k_total / oz::KT, oz::KT, c->sm_count, (double)rows_out * QW * 8.0,
                             (double)c->Np * c->Dp * c->npa);
  while (sp.per_split > oz::MAX_K_PER_ITEM || (size_t)sp.nsplit * rows_out * QW * 8 > cap) {
    if (sp.per_split > oz::MAX_K_PER_ITEM) sp.per_split = oz::MAX_K_PER_ITEM;
    else sp.per_split *= 2;
    sp.nsplit = (int)((k_total + sp.per_split - 1) / sp.per_split);
  }
  return sp;
}

template <int QW, int NPA>
int launch_persistent_t(cofem_ctx* c, double beta, int q_real, const cofem_cg_config* cg) {
  using PC = oz::PsCfg<QW, NPA>;
  static DeviceFlags flags;
  CKR(smem_attr_once(flags, oz::pcg_persistent<QW, NPA>, PC::SMEM));
  const int slot = QW / 8;
  if (!c->map_p_ok[slot]) {
    CKR(encode_u8_kblocked(&c->map_p[slot], c->pq, c->Dp, QW, QW));
    c->map_p_ok[slot] = true;
  }
  if (!c->map_v_ok[slot]) {
    CKR(encode_u8_kblocked(&c->map_v[slot], c->vq, c->Np, QW, QW));
    c->map_v_ok[slot] = true;
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, oz::pcg_persistent<QW, NPA>, oz::PS_THREADS, PC::SMEM));
  if (occ < 1) return fail(COFEM_ECUDA, "persistent PCG kernel cannot be resident");
  const int grid = c->sm_count;
  if ((size_t)grid * 4 * QW > (size_t)c->nblk_elem * 2 * std::max(c->ldq, QCHUNK))
    return fail(COFEM_ECUDA, "persistent PCG partials do not fit");
  const SplitPlan fp = persistent_splits(c, c->Np, c->Dp, c->vpart_cap, QW);
  const SplitPlan bp = persistent_splits(c, c->Dp, c->Np, c->ppart_cap, QW);
  // grid barrier words
  const size_t nbar = 2;
  if (c->gbar_cap < nbar) {
    if (c->gbar) cudaFree(c->gbar);
    c->gbar = nullptr;
    CK(cudaMalloc(&c->gbar, nbar * sizeof(unsigned)));
    c->gbar_cap = nbar;
  }
  CK(cudaMemsetAsync(c->gbar, 0, nbar * sizeof(unsigned), c->stream));
  unsigned long long* times = nullptr;
  if (c->time_kernels) {
    const int need = (cg->max_steps + 1) * oz::PS_TIMES;
    if (c->ptimes_cap < need) {
      if (c->ptimes) cudaFree(c->ptimes);
      c->ptimes = nullptr;
      CK(cudaMalloc(&c->ptimes, need * sizeof(unsigned long long)));
      c->ptimes_cap = need;
    }
    CK(cudaMemsetAsync(c->ptimes, 0, need * sizeof(unsigned long long), c->stream));
    times = c->ptimes;
  }
  Scalars sc = c->sc();
  oz::PcgPersistArgs a{};
  a.Np = c->Np;
  a.Dp = c->Dp;
  a.N = c->N;
  a.D = c->D;
  a.q_real = q_real;
  a.f_mblocks = (int)(c->Np / oz::BM);
  a.f_nsplit = fp.nsplit;
  a.f_kps = fp.per_split;
  a.f_items = a.f_mblocks * fp.nsplit;
  a.b_mblocks = (int)(c->Dp / oz::BM);
  a.b_nsplit = bp.nsplit;
  a.b_kps = bp.per_split;
  a.b_items = a.b_mblocks * bp.nsplit;
  a.rowscale = c->rowscale;
  a.colscale = c->colscale;
  a.P0 = (double*)c->P;
  a.P1 = (double*)c->P2;
  a.X = (double*)c->X;
  a.R = (double*)c->R;
  a.minv = c->minv;
  a.alpha = c->alpha;
  a.vpart = (double*)c->vpart;
  a.ppart = (double*)c->ppart;
  a.V = (double*)c->V;
  a.pq = c->pq;
  a.vq = c->vq;
  a.colmax_p = c->colmax;
  a.colmax_v = c->vcolmax;
  a.red = c->partials;
  a.rho1 = sc.rho[1];
  a.bn2 = sc.bn2;
  a.frozen = c->frozen;
  a.beta = beta;
  a.tol = cg->tolerance;
  a.max_steps = cg->max_steps;
  a.printed = cg->printed_recursion;
  a.st = c->st;
  a.bar = c->gbar;
  a.times = times;
  void* args[] = {&c->map_phi_fwd, &c->map_p[slot], &c->map_phiT, &c->map_v[slot], &a};
  cudaEvent_t e0 = nullptr;
  if (c->time_kernels) {
    e0 = next_event(c);
    cudaEventRecord(e0, c->stream);
  }
  CK(cudaLaunchCooperativeKernel((const void*)oz::pcg_persistent<QW, NPA>, dim3(grid), dim3(oz::PS_THREADS), args,
                                 PC::SMEM, c->stream));
  if (c->time_kernels) {
    cudaEvent_t e1 = next_event(c);
    cudaEventRecord(e1, c->stream);
    c->timed.push_back({2, c->evnext - 2});
  }
  c->launches++;
  c->solve_launches++;
  return 0;
}

int launch_persistent(cofem_ctx* c, double beta, int q_real, const cofem_cg_config* cg) {
  const bool p3 = c->npa == 3;
  switch (c->ldq) {
    case 8: return p3 ? launch_persistent_t<8, 3>(c, beta, q_real, cg) : launch_persistent_t<8, 4>(c, beta, q_real, cg);
    case 16: return p3 ? launch_persistent_t<16, 3>(c, beta, q_real, cg) : launch_persistent_t<16, 4>(c, beta, q_real, cg);
    case 24: return p3 ? launch_persistent_t<24, 3>(c, beta, q_real, cg) : launch_persistent_t<24, 4>(c, beta, q_real, cg);
    case 32: return p3 ? launch_persistent_t<32, 3>(c, beta, q_real, cg) : launch_persistent_t<32, 4>(c, beta, q_real, cg);
  }
  return fail(COFEM_EINVAL, "persistent PCG: unsupported column count");
}

// phase stamps of the last persistent solve -> contraction phase times
int persistent_phase_times(cofem_ctx* c, int steps) {
  if (!c->ptimes || steps < 1) return 0;
  std::vector<unsigned long long> t((size_t)(steps + 1) * oz::PS_TIMES);
  CK(cudaMemcpy(t.data(), c->ptimes, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  for (int u = 1; u <= steps; ++u) {
    const unsigned long long* s = &t[(size_t)u * oz::PS_TIMES];
    if (s[2] > s[1]) c->ph_fwd_ms += (s[2] - s[1]) * 1e-6;  // Phi P phase
    if (s[5] > s[4]) c->ph_bwd_ms += (s[5] - s[4]) * 1e-6;  // Phi^T V phase
  }
  if (getenv("COFEM_PHASE_DUMP") && steps > 1) {  // mean phase durations (us), steps 1..steps-1
    double ph[7] = {}, wk[7] = {};
    for (int u = 1; u < steps; ++u) {
      const unsigned long long* s = &t[(size_t)u * oz::PS_TIMES];
      const unsigned long long* n = &t[(size_t)(u + 1) * oz::PS_TIMES];
      for (int p = 0; p < 7; ++p) {
        ph[p] += ((p < 6 ? s[p + 1] : n[0]) - s[p]) * 1e-3;
        wk[p] += (s[8 + p] - s[p]) * 1e-3;
      }
    }
    const double m = 1.0 / (steps - 1);
    fprintf(stderr, "phases(us) A %.1f B %.1f C %.1f D %.1f E %.1f F %.1f H %.1f | CTA0 work A %.1f B %.1f C %.1f "
            "D %.1f E %.1f F %.1f H %.1f\n", ph[0] * m, ph[1] * m, ph[2] * m, ph[3] * m, ph[4] * m, ph[5] * m,
            ph[6] * m, wk[0] * m, wk[1] * m, wk[2] * m, wk[3] * m, wk[4] * m, wk[5] * m, wk[6] * m);
  }
  c->fwd_launches += steps;
  c->bwd_launches += steps;
  return 0;
}

// the blocked PCG on resident R (= B), minv, groups; result in X
template <typename T>
int pcg_device(cofem_ctx* c, double beta, int q_real, int ngroups, const int* groups, const cofem_cg_config* cg,
               cofem_cg_report* rep) {
  Scalars sc = c->sc();
  const int ldq = c->ldq;
  const int bs = elem_block(ldq);
  memset(rep, 0, sizeof(*rep));
  // device status reset; rho[0] = 1
  Status s0{};
  CK(cudaMemcpyAsync(c->st, &s0, sizeof(Status), cudaMemcpyHostToDevice, c->stream));
  std::vector<double> ones(ldq, 1.0);
  CK(cudaMemcpyAsync(sc.rho[0], ones.data(), ldq * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->frozen, 0, ldq * sizeof(int), c->stream));
  CK(cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c->stream));

  k_pcg_init<T><<<c->nblk_elem, bs, 2 * bs * sizeof(double), c->stream>>>(
      c->Dp, ldq, q_real, (T*)c->X, (T*)c->P, (const T*)c->R, c->minv, ngroups, groups, sc);
  c->launches++;
  CK(cudaGetLastError());
  CKR(allreduce(c, sc.bn2, ldq, ncclFloat64));
  CKR(allreduce(c, sc.rho_new, ldq, ncclFloat64));
  // entry checks (cg.py:116-122) need ||B||
  std::vector<double> bn2(ldq);
  CK(cudaMemcpyAsync(bn2.data(), sc.bn2, ldq * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  double b2 = 0;
  for (double v : bn2) b2 += v;
  const double bnorm = sqrt(b2);
  if (bnorm == 0.0) {
    rep->steps_taken = 0;
    rep->final_relative_residual = 0.0;
    rep->converged = 1;
    return 0;
  }
  if (1.0 <= cg->tolerance) {
    rep->steps_taken = 0;
    rep->final_relative_residual = 1.0;
    rep->converged = 1;
    return 0;
  }
  // ozaki: k_direction also emits the column maxima of diag(c) P for the next
  // Phi P quantisation (k_update re-zeroes them every step)
  const bool oz = c->prec == COFEM_OZAKI;
  if (oz && c->kind != 2) {
    if (c->kind == 0) CKR(ensure_oz(c));
    CK(cudaMemsetAsync(c->colmax, 0, ldq * sizeof(unsigned long long), c->stream));
  }
  unsigned long long* pmax = (oz && c->kind != 2) ? c->colmax : nullptr;
  const bool fused = std::is_same<T, double>::value && conv_fused_eligible(c, ngroups);
  const bool psifree = std::is_same<T, double>::value && dct_psifree_eligible(c);
  Scalars sc_asc = sc;  // the Psi-free step's direction kernel sweeps ascending (k_update_psi ends at the low rows)
  sc_asc.rev_rows = 0;
  if (fused) {
    // first direction P(1) = M^-1 B with its planes: the bound is max |M^-1 B| (max |P(0)| = 0)
    CK(cudaMemsetAsync(c->fz_max, 0, 4 * 32 * sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->vcolmax, 0, QCHUNK * sizeof(unsigned long long), c->stream));
    const int cbs = ldq * (256 / ldq);
    oz::k_colmax<double><<<2 * c->sm_count, cbs, cbs * sizeof(double), c->stream>>>(
        c->D, ldq, 0, ldq, (const double*)c->R, cg->printed_recursion ? nullptr : c->minv, c->fz_max + 64, c->st);
    c->launches++;
    CKR(conv_fused(c, 3, 0, beta, q_real, cg));
  } else if (psifree) {
    k_pap_init<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
        c->Dp, ldq, q_real, cg->printed_recursion, (const T*)c->R, c->alpha, c->minv, ngroups, groups, c->dct_fscal,
        c->dct_partials4, sc);
    k_direction<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
        c->Dp, ldq, q_real, 0, cg->max_steps, cg->tolerance, cg->printed_recursion, (T*)c->P, (const T*)c->R, c->minv,
        ngroups, groups, sc_asc, c->colscale, pmax, c->st);
    c->launches += 2;
  } else {
    k_direction<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
        c->Dp, ldq, q_real, 0, cg->max_steps, cg->tolerance, cg->printed_recursion, (T*)c->P, (const T*)c->R, c->minv,
        ngroups, groups, sc, c->colscale, pmax, c->st);
    c->launches++;
  }
  CK(cudaGetLastError());
  c->p_colmax_valid = oz;

  const bool persistent = std::is_same<T, double>::value && persistent_eligible(c, ngroups);
  if (persistent) CKR(launch_persistent(c, beta, q_real, cg));
  int u = 1;
  for (; !persistent && u <= cg->max_steps; ++u) {
    if (u > LAG) {
      const int slot = (u - LAG) % LAG;
      CK(cudaEventSynchronize(c->ev[slot]));
      if (c->h_st[slot].done) break;
    }
    if (fused) {
      const int slot = u % LAG;
      CKR(conv_fused(c, 0, u, beta, q_real, cg));
      CKR(conv_fused(c, 1, u, beta, q_real, cg));
      CKR(conv_fused(c, 2, u, beta, q_real, cg));
      CKR(conv_fused(c, 3, u, beta, q_real, cg, c->d_hst + slot));
      std::swap(c->P, c->P2);
      CK(cudaEventRecord(c->ev[slot], c->stream));
      continue;
    }
    if (psifree) {
      const int slot = u % LAG;
      CKR(dct_apply_vv(c, c->st));
      k_update_psi<T><<<c->nblk_elem, bs, 4 * bs * sizeof(double), c->stream>>>(
          c->Dp, ldq, q_real, u, cg->printed_recursion, (T*)c->R, (const T*)c->P, (const T*)c->bufA, beta, c->alpha,
          c->minv, ngroups, groups, c->dct_partials, c->dct_vv_blocks, c->dct_fscal, c->dct_partials4, sc, c->st);
      c->launches++;
      tick(c, 4);
      k_direction<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
          c->Dp, ldq, q_real, u, cg->max_steps, cg->tolerance, cg->printed_recursion, (T*)c->P, (const T*)c->R,
          c->minv, ngroups, groups, sc_asc, c->colscale, pmax, c->st, nullptr, c->d_hst + slot, (T*)c->X, (T*)c->P2,
          (const T*)c->P2);
      std::swap(c->P, c->P2);
      c->launches++;
      tick(c, 5);
      CK(cudaGetLastError());
      CK(cudaEventRecord(c->ev[slot], c->stream));
      continue;
    }
    CKR(system_apply_dev<T>(c, beta, c->st));
    CKR(allreduce(c, sc.pi, ldq, ncclFloat64));
    k_update<T><<<c->nblk_elem, bs, 2 * bs * sizeof(double), c->stream>>>(
        c->Dp, ldq, q_real, u & 1, nullptr, (T*)c->R, (const T*)c->P, (const T*)c->Psi, c->minv, ngroups, groups,
        sc, pmax, c->st);
    c->launches++;
    tick(c, 4);
    CK(cudaGetLastError());
    CKR(allreduce(c, sc.rho_new, 2 * ldq, ncclFloat64));  // rho_new | rn2
    const int slot = u % LAG;
    // the kernel mirrors the status into the host-mapped slot: no copy in the stream
    k_direction<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(
        c->Dp, ldq, q_real, u, cg->max_steps, cg->tolerance, cg->printed_recursion, (T*)c->P, (const T*)c->R,
        c->minv, ngroups, groups, sc, c->colscale, pmax, c->st, nullptr, c->d_hst + slot, (T*)c->X, (T*)c->P2,
        (const T*)c->P2);
    std::swap(c->P, c->P2);  // P(u+1) is the next step's direction
    c->launches++;
    tick(c, 5);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[slot], c->stream));
  }
  c->p_colmax_valid = false;
  Status fin;
  CK(cudaMemcpyAsync(&fin, c->st, sizeof(Status), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->pcg_steps += fin.steps;
  if (persistent && c->time_kernels) CKR(persistent_phase_times(c, fin.steps));
  rep->steps_taken = fin.steps;
  rep->converged = fin.converged;
  rep->diverged = fin.diverged;
  rep->final_relative_residual = fin.delta;
  std::vector<int> fz(ldq);
  CK(cudaMemcpy(fz.data(), c->frozen, ldq * sizeof(int), cudaMemcpyDeviceToHost));
  int nb = 0;
  for (int q = 0; q < q_real; ++q) nb += fz[q] ? 1 : 0;
  rep->n_breakdown = nb;
  if (fin.diverged) return fail(COFEM_EDIVERGED, "non-finite residual at CG step " + std::to_string(fin.steps));
  return 0;
}

// ---- multi-task lockstep PCG (cg.solve_blocked over the tasks' systems,
// cg.py:201-234, as run_cofem_multitask drives it): every task keeps its own
// blocks and per-column scalars; the stopping rule aggregates ||R||_F and
// ||B||_F over all tasks (k_sum_tasks -> agg), and one status gates them all.
// All contexts run on task 0's stream.
template <typename T>
int pcg_multi(cofem_ctx** cs, int L, const double* betas, int q_real, const cofem_cg_config* cg, cofem_cg_report* rep,
              double* agg, double** dptrs) {
  cofem_ctx* c0 = cs[0];
  const int ldq = c0->ldq;
  const int bs = elem_block(ldq);
  memset(rep, 0, sizeof(*rep));
  Status s0{};
  Status* st = c0->st;
  CK(cudaMemcpyAsync(st, &s0, sizeof(Status), cudaMemcpyHostToDevice, c0->stream));
  std::vector<double> ones(ldq, 1.0);
  // pointer tables: rn2[L] | bn2[L]
  std::vector<double*> tab(2 * L);
  for (int l = 0; l < L; ++l) {
    cofem_ctx* c = cs[l];
    Scalars sc = c->sc();
    tab[l] = sc.rn2;
    tab[L + l] = sc.bn2;
    CK(cudaMemcpyAsync(sc.rho[0], ones.data(), ldq * sizeof(double), cudaMemcpyHostToDevice, c0->stream));
    CK(cudaMemsetAsync(c->frozen, 0, ldq * sizeof(int), c0->stream));
    CK(cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c0->stream));
    k_pcg_init<T><<<c->nblk_elem, bs, 2 * bs * sizeof(double), c0->stream>>>(
        c->Dp, ldq, q_real, (T*)c->X, (T*)c->P, (const T*)c->R, c->minv, 1, nullptr, sc);
    c->launches++;
  }
  CK(cudaMemcpyAsync(dptrs, tab.data(), 2 * L * sizeof(double*), cudaMemcpyHostToDevice, c0->stream));
  k_sum_tasks<<<1, 1, 0, c0->stream>>>(L, ldq, (const double* const*)dptrs, (const double* const*)(dptrs + L), agg);
  CK(cudaGetLastError());
  double hagg[2];
  CK(cudaMemcpyAsync(hagg, agg, 2 * sizeof(double), cudaMemcpyDeviceToHost, c0->stream));
  CK(cudaStreamSynchronize(c0->stream));
  const double bnorm = sqrt(hagg[1]);
  if (bnorm == 0.0) {
    rep->converged = 1;
    return 0;
  }
  if (1.0 <= cg->tolerance) {
    rep->final_relative_residual = 1.0;
    rep->converged = 1;
    return 0;
  }
  const bool oz = c0->prec == COFEM_OZAKI;
  for (int l = 0; l < L; ++l) {
    cofem_ctx* c = cs[l];
    const bool fused = oz && c->kind != 2;
    if (fused) {
      if (c->kind == 0) CKR(ensure_oz(c));
      CK(cudaMemsetAsync(c->colmax, 0, ldq * sizeof(unsigned long long), c0->stream));
    }
    k_direction<T><<<c->nblk_elem, bs, bs * sizeof(double), c0->stream>>>(
        c->Dp, ldq, q_real, 0, cg->max_steps, cg->tolerance, cg->printed_recursion, (T*)c->P, (const T*)c->R,
        c->minv, 1, nullptr, c->sc(), c->colscale, fused ? c->colmax : nullptr, st, agg);
    c->launches++;
    c->p_colmax_valid = fused;
  }
  CK(cudaGetLastError());
  int u = 1;
  for (; u <= cg->max_steps; ++u) {
    if (u > LAG) {
      const int slot = (u - LAG) % LAG;
      CK(cudaEventSynchronize(c0->ev[slot]));
      if (c0->h_st[slot].done) break;
    }
    for (int l = 0; l < L; ++l) {
      cofem_ctx* c = cs[l];
      const bool fused = oz && c->kind != 2;
      CKR(system_apply_dev<T>(c, betas[l], st));
      k_update<T><<<c->nblk_elem, bs, 2 * bs * sizeof(double), c0->stream>>>(
          c->Dp, ldq, q_real, u & 1, nullptr, (T*)c->R, (const T*)c->P, (const T*)c->Psi, c->minv, 1, nullptr,
          c->sc(), fused ? c->colmax : nullptr, st);
      c->launches++;
    }
    k_sum_tasks<<<1, 1, 0, c0->stream>>>(L, ldq, (const double* const*)dptrs, (const double* const*)(dptrs + L), agg);
    const int slot = u % LAG;
    for (int l = 0; l < L; ++l) {
      cofem_ctx* c = cs[l];
      const bool fused = oz && c->kind != 2;
      k_direction<T><<<c->nblk_elem, bs, bs * sizeof(double), c0->stream>>>(
          c->Dp, ldq, q_real, u, cg->max_steps, cg->tolerance, cg->printed_recursion, (T*)c->P, (const T*)c->R,
          c->minv, 1, nullptr, c->sc(), c->colscale, fused ? c->colmax : nullptr, st, agg,
          l == L - 1 ? c0->d_hst + slot : nullptr, (T*)c->X, (T*)c->P2, (const T*)c->P2);
      std::swap(c->P, c->P2);
      c->launches++;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c0->ev[slot], c0->stream));
  }
  for (int l = 0; l < L; ++l) cs[l]->p_colmax_valid = false;
  Status fin;
  CK(cudaMemcpyAsync(&fin, st, sizeof(Status), cudaMemcpyDeviceToHost, c0->stream));
  CK(cudaStreamSynchronize(c0->stream));
  c0->pcg_steps += fin.steps;
  rep->steps_taken = fin.steps;
  rep->converged = fin.converged;
  rep->diverged = fin.diverged;
  rep->final_relative_residual = fin.delta;
  if (fin.diverged) return fail(COFEM_EDIVERGED, "non-finite residual at CG step " + std::to_string(fin.steps));
  return 0;
}

// host double (rows x q, row stride q) -> device T (rows_pad x ldq, zero padded)
template <typename T>
int upload_block(cofem_ctx* c, const double* h, int64_t rows, int64_t q, int64_t rows_pad, int ldq, void* dst) {
  std::vector<T> tmp((size_t)rows_pad * ldq, T(0));
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t k = 0; k < q; ++k) tmp[i * ldq + k] = (T)h[i * q + k];
  CK(cudaMemcpyAsync(dst, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

// Host -> device upload of a pitched row block from pageable memory: host
// threads copy row chunks into two pinned staging buffers while the copy
// engine drains the other one (pageable cudaMemcpy stages through one driver
// buffer at ~11 GB/s; this runs at the PCIe rate).
// the staging buffers (2 x 64 MB) are pinned once per process and reused:
// page-locking them costs ~70 ms, the upload of a 4.3 GB dictionary then runs
// at ~42 GB/s; one upload at a time
struct PinnedPool {
  std::mutex m;
  void* buf[2] = {nullptr, nullptr};
  size_t bytes = 0;
};
PinnedPool g_pin;

int upload_rows(cofem_ctx* c, void* dst, size_t dpitch, const void* src, size_t spitch, size_t row_bytes,
                int64_t rows) {
  constexpr size_t CHUNK = (size_t)64 << 20;
  if ((size_t)rows * row_bytes < 2 * CHUNK) {  // small: one pageable copy
    CK(cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyHostToDevice, c->stream));
    return 0;
  }
  const int64_t rpc = std::max<int64_t>(1, (int64_t)(CHUNK / row_bytes));
  std::lock_guard<std::mutex> lk(g_pin.m);
  if (g_pin.bytes < (size_t)rpc * row_bytes) {
    for (int b = 0; b < 2; ++b)
      if (g_pin.buf[b]) cudaFreeHost(g_pin.buf[b]);
    g_pin.buf[0] = g_pin.buf[1] = nullptr;
    g_pin.bytes = 0;
    for (int b = 0; b < 2; ++b)
      if (cudaHostAlloc(&g_pin.buf[b], (size_t)rpc * row_bytes, cudaHostAllocPortable) != cudaSuccess)
        return fail(COFEM_ENOMEM, "pinned staging buffers");
    g_pin.bytes = (size_t)rpc * row_bytes;
  }
  void* pin[2] = {g_pin.buf[0], g_pin.buf[1]};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int rc = 0;
  for (int b = 0; b < 2 && !rc; ++b) {
    if (cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess)
      rc = fail(COFEM_ECUDA, "staging events");
  }
  const int nthr = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (int64_t r0 = 0, i = 0; r0 < rows && !rc; r0 += rpc, ++i) {
    const int b = (int)(i & 1);
    const int64_t nr = std::min(rpc, rows - r0);
    if (i >= 2 && cudaEventSynchronize(ev[b]) != cudaSuccess) rc = fail(COFEM_ECUDA, "staging event");
    if (rc) break;
    auto copy = [&](int t) {
      for (int64_t r = r0 + t; r < r0 + nr; r += nthr)
        memcpy((char*)pin[b] + (size_t)(r - r0) * row_bytes, (const char*)src + (size_t)r * spitch, row_bytes);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nthr; ++t) pool.emplace_back(copy, t);
    copy(0);
    for (auto& th : pool) th.join();
    if (cudaMemcpy2DAsync((char*)dst + (size_t)r0 * dpitch, dpitch, pin[b], row_bytes, row_bytes, nr,
                          cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        cudaEventRecord(ev[b], c->stream) != cudaSuccess)
      rc = fail(COFEM_ECUDA, "staged upload");
  }
  cudaStreamSynchronize(c->stream);
  for (int b = 0; b < 2; ++b)
    if (ev[b]) cudaEventDestroy(ev[b]);
  return rc;
}

// Device -> host download of a pitched row block into packed pageable rows, the mirror of
// upload_rows: the copy engine fills one pinned staging buffer (rows packed by the 2-D copy)
// while host threads move the other one into the caller's buffer -- a fresh numpy array is
// untouched memory, and one thread taking its page faults ran a 1 GB block at 1.4 GB/s.
int download_rows(cofem_ctx* c, void* dst, const void* src, size_t spitch, size_t row_bytes, int64_t rows) {
  // 16 MB chunks: when no dictionary upload has pinned the pool yet, page-locking 2 x 64 MB
  // (~70 ms) would cost more than the download itself
  constexpr size_t CHUNK = (size_t)16 << 20;
  const int64_t rpc = std::max<int64_t>(1, (int64_t)(CHUNK / row_bytes));
  std::lock_guard<std::mutex> lk(g_pin.m);
  if (g_pin.bytes < (size_t)rpc * row_bytes) {
    for (int b = 0; b < 2; ++b)
      if (g_pin.buf[b]) cudaFreeHost(g_pin.buf[b]);
    g_pin.buf[0] = g_pin.buf[1] = nullptr;
    g_pin.bytes = 0;
    for (int b = 0; b < 2; ++b)
      if (cudaHostAlloc(&g_pin.buf[b], (size_t)rpc * row_bytes, cudaHostAllocPortable) != cudaSuccess)
        return fail(COFEM_ENOMEM, "pinned staging buffers");
    g_pin.bytes = (size_t)rpc * row_bytes;
  }
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b)
    if (cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess) return fail(COFEM_ECUDA, "staging events");
  const int nthr = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const int64_t nchunks = (rows + rpc - 1) / rpc;
  int rc = 0;
  auto issue = [&](int64_t i) {
    const int b = (int)(i & 1);
    const int64_t r0 = i * rpc, nr = std::min(rpc, rows - r0);
    if (cudaMemcpy2DAsync(g_pin.buf[b], row_bytes, (const char*)src + (size_t)r0 * spitch, spitch, row_bytes, nr,
                          cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaEventRecord(ev[b], c->stream) != cudaSuccess)
      rc = fail(COFEM_ECUDA, "staged download");
  };
  issue(0);
  for (int64_t i = 0; i < nchunks && !rc; ++i) {
    const int b = (int)(i & 1);
    const int64_t r0 = i * rpc, nr = std::min(rpc, rows - r0);
    if (i + 1 < nchunks) issue(i + 1);  // the other buffer: its previous contents were consumed in trip i - 1
    if (rc) break;
    if (cudaEventSynchronize(ev[b]) != cudaSuccess) {
      rc = fail(COFEM_ECUDA, "staging event");
      break;
    }
    const size_t total = (size_t)nr * row_bytes;
    char* out = (char*)dst + (size_t)r0 * row_bytes;
    const char* in = (const char*)g_pin.buf[b];
    auto copy = [&](int t) {
      const size_t per = (total / nthr + 4095) & ~(size_t)4095;
      const size_t a = std::min(total, (size_t)t * per), e = std::min(total, a + per);
      if (e > a) memcpy(out + a, in + a, e - a);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nthr; ++t) pool.emplace_back(copy, t);
    copy(0);
    for (auto& th : pool) th.join();
  }
  cudaStreamSynchronize(c->stream);
  for (int b = 0; b < 2; ++b)
    if (ev[b]) cudaEventDestroy(ev[b]);
  return rc;
}

template <typename T>
int download_block(cofem_ctx* c, const void* src, int64_t rows, int64_t q, int ldq, int qoff, double* h) {
  if (std::is_same<T, double>::value && (size_t)rows * q * sizeof(double) >= ((size_t)32 << 20))
    return download_rows(c, h, (const double*)src + qoff, (size_t)ldq * sizeof(double), (size_t)q * sizeof(double), rows);
  std::vector<T> tmp((size_t)rows * ldq);
  CK(cudaMemcpyAsync(tmp.data(), src, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t k = 0; k < q; ++k) h[i * q + k] = (double)tmp[i * ldq + qoff + k];
  return 0;
}

int check_ctx(cofem_ctx* c, bool need_phi = true) {
  if (!c) return fail(COFEM_EINVAL, "null context");
  if (need_phi && !c->have_phi) return fail(COFEM_ESTATE, "no dictionary set");
  return set_dev(c);
}

int ldq_for(int64_t q) { return (int)round_up(std::max<int64_t>(q, 1), 8); }

// column squared norms of a dense dictionary (the exact float64 copy when held)
int dense_colsq(cofem_ctx* c) {
  const int g = (int)((c->D + 255) / 256);
  if (c->phi64) k_colsq<double><<<g, 256, 0, c->stream>>>(c->phi64, c->Dp, c->N, c->D, c->colsq);
  else k_colsq<float><<<g, 256, 0, c->stream>>>(c->phi, c->Dp, c->N, c->D, c->colsq);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// ---- apply / adjoint / system apply ---------------------------------------
// DCT: tmpD (D x ldq) <- Phi^T V for V (N x ldq) already in c->V
int dct_adjoint_from_V(cofem_ctx* c) {
  const int64_t n = c->dct_n, ldq = c->ldq;
  CK(cudaMemsetAsync(c->bufB, 0, (size_t)n * n * ldq * sizeof(double), c->stream));
  dctf::k_scatter<<<8 * c->sm_count, 256, 0, c->stream>>>(c->N, (int)ldq, c->dct_mask, (const double*)c->V,
                                                          c->bufB);
  c->launches++;
  return dct_adjoint_dev(c, (double*)c->tmpD, nullptr);
}

template <typename T>
int apply_impl(cofem_ctx* c, const double* V, int64_t q, double* out) {
  const int ldq = ldq_for(q);
  CKR(ensure_ws(c, ldq));
  CKR(upload_block<T>(c, V, c->D, q, c->Dp, ldq, c->P));
  if (c->conv_fft) {
    CKR(conv_fft_pass(c, (const double*)c->P, (double*)c->V, false, nullptr));
    return download_block<T>(c, c->V, c->N, q, ldq, 0, out);
  }
  if (c->kind == 3) {
    CKR(dct1_inverse(c, (const double*)c->P));
    dct1::k_gather<<<8 * c->sm_count, 256, 0, c->stream>>>(c->N, c->Np, c->D, ldq, c->dct_mask,
                                                           reinterpret_cast<const double2*>(c->bufA), (double*)c->V);
    c->launches++;
    CK(cudaGetLastError());
    return download_block<T>(c, c->V, c->N, q, ldq, 0, out);
  }
  if (c->kind == 2) {
    CKR(dct_forward_dev(c, (const double*)c->P, nullptr));
    dctf::k_gather<<<8 * c->sm_count, 256, 0, c->stream>>>(c->N, ldq, c->dct_mask, c->bufB, (double*)c->V);
    c->launches++;
    CK(cudaGetLastError());
    return download_block<T>(c, c->V, c->N, q, ldq, 0, out);
  }
  std::vector<double> chunk;
  for (int qoff = 0; qoff < ldq; qoff += QCHUNK) {
    const int qpc = chunk_width(ldq, qoff);
    CKR(fwd_chunk<T>(c, qpc, (const T*)c->P, ldq, qoff, (T*)c->V, nullptr));
    CKR(reduce_partial_v(c, (size_t)c->Np * qpc, nccl_t<T>()));
    const int64_t qn = std::min<int64_t>(qpc, q - qoff);
    if (qn <= 0) break;
    chunk.assign((size_t)c->N * qn, 0.0);
    CKR(download_block<T>(c, c->V, c->N, qn, qpc, 0, chunk.data()));
    for (int64_t i = 0; i < c->N; ++i)
      for (int64_t k = 0; k < qn; ++k) out[i * q + qoff + k] = chunk[i * qn + k];
  }
  return 0;
}

template <typename T>
int adjoint_impl(cofem_ctx* c, const double* U, int64_t q, double* out) {
  const int ldq = ldq_for(q);
  CKR(ensure_ws(c, ldq));
  if (c->conv_fft) {
    CKR(upload_block<T>(c, U, c->N, q, c->Np, ldq, c->V));
    CKR(conv_fft_pass(c, (const double*)c->V, (double*)c->tmpD, true, nullptr));
    return download_block<T>(c, c->tmpD, c->D, q, ldq, 0, out);
  }
  if (c->kind == 2 || c->kind == 3) {
    CKR(upload_block<T>(c, U, c->N, q, c->Np, ldq, c->V));
    CKR(c->kind == 2 ? dct_adjoint_from_V(c) : dct1_adjoint_from_V(c));
    return download_block<T>(c, c->tmpD, c->D, q, ldq, 0, out);
  }
  std::vector<double> chunk;
  for (int qoff = 0; qoff < ldq; qoff += QCHUNK) {
    const int qpc = chunk_width(ldq, qoff);
    const int64_t qn = std::min<int64_t>(qpc, q - qoff);
    if (qn <= 0) break;
    // gather columns [qoff, qoff+qn) of U into a dense Np x qpc block
    std::vector<double> sub((size_t)c->N * qn);
    for (int64_t i = 0; i < c->N; ++i)
      for (int64_t k = 0; k < qn; ++k) sub[i * qn + k] = U[i * q + qoff + k];
    CKR(upload_block<T>(c, sub.data(), c->N, qn, c->Np, qpc, c->V));
    c->v_colmax_valid = false;
    int ns = 1;
    CKR(bwd_chunk<T>(c, qpc, (const T*)c->V, &ns, nullptr));
    const int bs = elem_block(qpc);
    k_sum_splits<T><<<c->nblk_elem, bs, bs * sizeof(double), c->stream>>>(c->Dp, qpc, ns, (const T*)c->ppart,
                                                                          (T*)c->tmpD, nullptr, nullptr, nullptr);
    c->launches++;
    CK(cudaGetLastError());
    chunk.assign((size_t)c->D * qn, 0.0);
    CKR(download_block<T>(c, c->tmpD, c->D, qn, qpc, 0, chunk.data()));
    for (int64_t j = 0; j < c->D; ++j)
      for (int64_t k = 0; k < qn; ++k) out[j * q + qoff + k] = chunk[j * qn + k];
  }
  return 0;
}

template <typename T>
int system_apply_impl(cofem_ctx* c, double beta, const double* alpha, const double* V, int64_t q, double* out) {
  const int ldq = ldq_for(q);
  CKR(ensure_ws(c, ldq));
  std::vector<double> a(c->Dp, 0.0);
  std::copy(alpha, alpha + c->D, a.begin());
  CK(h2d_sync(c, c->alpha, a.data(), c->Dp * sizeof(double)));
  CKR(upload_block<T>(c, V, c->D, q, c->Dp, ldq, c->P));
  CK(cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c->stream));
  CKR(system_apply_dev<T>(c, beta, nullptr));
  CKR(download_block<T>(c, c->Psi, c->D, q, ldq, 0, out));
  return 0;
}

// ---- EM loop ---------------------------------------------------------------
template <typename T>
int compute_aty(cofem_ctx* c, const double* y_host) {
  // V[:, 0] = y, other columns 0 -> Phi^T V (structured: all ldq columns of
  // the passes; dense / band: the 8-wide bwd contraction); aty = column 0.
  // y goes up as N doubles and aty is gathered on the device (no host
  // staging of the Np x ldq blocks).
  CKR(ensure_ws(c, std::max(c->ldq, 8)));
  const bool whole = c->kind == 2 || c->kind == 3 || c->conv_fft;
  const int ld = whole ? c->ldq : 8;
  if (!c->ybuf) CK(cudaMalloc(&c->ybuf, c->Np * sizeof(double)));
  CK(cudaMemcpyAsync(c->ybuf, y_host, c->N * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const int g = 8 * c->sm_count;
  if (whole) {
    k_put_col0<double><<<g, 256, 0, c->stream>>>(c->ybuf, c->N, c->Np, ld, (double*)c->V);
    c->launches++;
    if (c->conv_fft) CKR(conv_fft_pass(c, (const double*)c->V, (double*)c->tmpD, true, nullptr));
    else if (c->kind == 3) CKR(dct1_adjoint_from_V(c));
    else CKR(dct_adjoint_from_V(c));
    k_get_col0<double><<<g, 256, 0, c->stream>>>((const double*)c->tmpD, c->D, c->Dp, ld, c->aty);
    c->launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    return 0;
  }
  k_put_col0<T><<<g, 256, 0, c->stream>>>(c->ybuf, c->N, c->Np, 8, (T*)c->V);
  c->launches++;
  c->v_colmax_valid = false;
  int ns = 1;
  CKR(bwd_chunk<T>(c, 8, (const T*)c->V, &ns, nullptr));
  const int bsz = elem_block(8);
  k_sum_splits<T><<<c->nblk_elem, bsz, bsz * sizeof(double), c->stream>>>(c->Dp, 8, ns, (const T*)c->ppart,
                                                                           (T*)c->tmpD, nullptr, nullptr, nullptr);
  c->launches++;
  k_get_col0<T><<<g, 256, 0, c->stream>>>((const T*)c->tmpD, c->D, c->Dp, 8, c->aty);
  c->launches++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int ensure_em_buffers(cofem_ctx* c, int K) {
  if (c->probes) cudaFree(c->probes);
  if (c->probe_store) cudaFree(c->probe_store);
  CK(cudaMalloc(&c->probes, (size_t)c->Dp * K));
  CK(cudaMalloc(&c->probe_store, (size_t)c->Dp * K));
  return 0;
}

template <typename T>
int em_prepare(cofem_ctx* c, const double* y, double beta, const cofem_em_config* em, const double* theta) {
  const int K = em->probes;
  const int ldq = ldq_for(K + 1);
  CKR(ensure_ws(c, ldq));
  CKR(ensure_em_buffers(c, K));
  CKR(compute_aty<T>(c, y));
  // alpha = 1 (PrecisionState.initial, cofem.py:65), theta by policy
  std::vector<double> a(c->Dp, 1.0);
  CK(h2d_sync(c, c->alpha, a.data(), c->Dp * sizeof(double)));
  if (em->theta_policy == COFEM_THETA_JACOBI) {
    if (c->kind == 2 || c->kind == 3)
      return fail(COFEM_EINVAL, "jacobi on a DCT dictionary: pass its column norms as custom theta");
    if (c->kind == 0) {
      CKR(dense_colsq(c));
    }
    CK(cudaMemcpyAsync(c->theta, c->colsq, c->D * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  } else if (em->theta_policy == COFEM_THETA_CUSTOM) {
    if (!theta) return fail(COFEM_EINVAL, "custom theta policy needs a theta vector");
    CK(h2d_sync(c, c->theta, theta, c->D * sizeof(double)));
  }
  k_make_minv<<<(int)((c->Dp + 255) / 256), 256, 0, c->stream>>>(c->D, c->Dp, beta, c->alpha, c->theta,
                                                                   em->theta_policy, c->minv);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

// EM iteration t's draw of the reference probe stream, this shard's rows, into c->probes
void draw_stream_probes(cofem_ctx* c, int t, int K) {
  const uint64_t stride = c->pcg_stride ? c->pcg_stride : (uint64_t)c->global_cols * K;  // 32-bit halves
  const int64_t nchunk = ((int64_t)c->D * K + 65) / 64 + 1;
  k_pcg64_rademacher<<<(int)std::min<int64_t>((nchunk + 255) / 256, 8 * c->sm_count), 256, 0, c->stream>>>(
      c->pcg_state[0], c->pcg_state[1], c->pcg_inc[0], c->pcg_inc[1], c->pcg_first + (uint64_t)(t - 1) * stride,
      c->col_offset, c->D, K, c->probes);
  c->launches++;
}

template <typename T>
int em_iteration(cofem_ctx* c, int t, int T_total, double beta, const cofem_em_config* em,
                 const cofem_cg_config* cg, const int8_t* probes_host_iter, uint64_t dseed, cofem_cg_report* rep) {
  const int K = em->probes;
  const int ldq = c->ldq;
  if (probes_host_iter) {
    CK(cudaMemcpyAsync(c->probes, probes_host_iter, (size_t)c->D * K, cudaMemcpyHostToDevice, c->stream));
  } else if (c->pcg_stream) {
    draw_stream_probes(c, t, K);
    probes_host_iter = c->probes;  // (only tested for non-null below)
  }
  const int bs = 256;
  const int64_t n = c->Dp * ldq;
  k_build_rhs<T><<<(int)std::min<int64_t>((n + bs - 1) / bs, 8 * c->sm_count), bs, 0, c->stream>>>(
      c->D, c->Dp, ldq, K, probes_host_iter ? c->probes : nullptr, dseed, t, c->col_offset, c->aty, (T*)c->R,
      c->probe_store);
  c->launches++;
  CK(cudaGetLastError());
  int rc = pcg_device<T>(c, beta, K + 1, 1, nullptr, cg, rep);
  if (rc != 0) return rc;
  const int do_update = t < T_total ? 1 : 0;
  k_em_finish<T><<<(int)((c->D + 255) / 256), 256, 0, c->stream>>>(
      c->D, ldq, K, beta, (const T*)c->X, c->probe_store, c->mu, c->s, c->alpha, c->minv, c->theta,
      em->theta_policy, do_update, em->variant, em->floor_eps, em->clamp_max);
  c->launches++;
  CK(cudaGetLastError());
  return 0;
}

template <typename T>
int run_impl(cofem_ctx* c, const double* y, double beta, const cofem_em_config* em, const cofem_cg_config* cg,
             const double* theta, const int8_t* probes, uint64_t dseed, double* alpha, double* mu, double* s,
             int32_t* steps, double* resid, int32_t* fail_it, int32_t* fail_step) {
  CKR(em_prepare<T>(c, y, beta, em, theta));
  std::vector<double> alpha_used(c->D, 1.0);
  c->run_wall.assign(em->iterations, 0.0);
  c->run_K = 0;
  for (int t = 1; t <= em->iterations; ++t) {
    const auto w0 = std::chrono::steady_clock::now();
    cofem_cg_report rep;
    // alpha of this E-step is what the caller gets back after the last one
    if (t == em->iterations && alpha) {
      CK(cudaMemcpyAsync(alpha_used.data(), c->alpha, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    const int8_t* pt = probes ? probes + (size_t)(t - 1) * c->D * em->probes : nullptr;
    int rc = em_iteration<T>(c, t, em->iterations, beta, em, cg, pt, dseed, &rep);
    if (steps) steps[t - 1] = rep.steps_taken;
    if (resid) resid[t - 1] = rep.final_relative_residual;
    if (rc == COFEM_EDIVERGED) {
      if (fail_it) *fail_it = t;
      if (fail_step) *fail_step = rep.steps_taken;
      return fail(COFEM_EDIVERGED, "non-finite residual at CG step " + std::to_string(rep.steps_taken) +
                                       " (EM iteration " + std::to_string(t) + ")");
    }
    if (rc != 0) return rc;
    c->run_rep = rep;
    if (t == em->iterations) CK(cudaStreamSynchronize(c->stream));  // the last M-step-free finish
    c->run_wall[t - 1] = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  }
  CK(cudaStreamSynchronize(c->stream));
  c->run_K = em->probes;
  if (alpha) std::copy(alpha_used.begin(), alpha_used.end(), alpha);
  if (mu) CK(cudaMemcpy(mu, c->mu, c->D * sizeof(double), cudaMemcpyDeviceToHost));
  if (s) CK(cudaMemcpy(s, c->s, c->D * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

// run_cofem_multitask (cofem.py:160-214): shared alpha, all L (K+1)-column
// systems in one lockstep PCG per EM iteration, pooled M-step
template <typename T>
int run_multi_impl(cofem_ctx** cs, int L, const double* const* ys, const double* betas, const cofem_em_config* em,
                   const cofem_cg_config* cg, const double* theta, const int8_t* probes, double* alpha,
                   double* const* mus, double* const* ss, int32_t* steps, double* resid, int32_t* fail_it,
                   int32_t* fail_step) {
  cofem_ctx* c0 = cs[0];
  const int K = em->probes;
  std::vector<cudaStream_t> saved(L);
  for (int l = 0; l < L; ++l) {
    saved[l] = cs[l]->stream;
    CKR(em_prepare<T>(cs[l], ys[l], betas[l], em, theta ? theta + (size_t)l * cs[l]->D : nullptr));
  }
  CK(cudaDeviceSynchronize());
  for (int l = 0; l < L; ++l) cs[l]->stream = c0->stream;  // one stream for the lockstep
  double* agg = nullptr;
  double** dptrs = nullptr;
  double** aptrs = nullptr;  // mu | s | alpha | minv | theta (L each)
  double* dbeta = nullptr;
  int rc = 0;
  auto cleanup = [&]() {
    for (int l = 0; l < L; ++l) cs[l]->stream = saved[l];
    if (agg) cudaFree(agg);
    if (dptrs) cudaFree(dptrs);
    if (aptrs) cudaFree(aptrs);
    if (dbeta) cudaFree(dbeta);
  };
  if (cudaMalloc(&agg, 2 * sizeof(double)) || cudaMalloc(&dptrs, 2 * L * sizeof(double*)) ||
      cudaMalloc(&aptrs, 5 * L * sizeof(double*)) || cudaMalloc(&dbeta, L * sizeof(double))) {
    cleanup();
    return fail(COFEM_ENOMEM, "multitask tables");
  }
  std::vector<double*> at(5 * L);
  for (int l = 0; l < L; ++l) {
    at[l] = cs[l]->mu;
    at[L + l] = cs[l]->s;
    at[2 * L + l] = cs[l]->alpha;
    at[3 * L + l] = cs[l]->minv;
    at[4 * L + l] = cs[l]->theta;
  }
  h2d_sync(c0, aptrs, at.data(), at.size() * sizeof(double*));
  h2d_sync(c0, dbeta, betas, L * sizeof(double));
  const int64_t dk = c0->D * K;
  for (int t = 1; t <= em->iterations && !rc; ++t) {
    for (int l = 0; l < L; ++l) {
      cofem_ctx* c = cs[l];
      if (probes) {
        const int8_t* pt = probes + ((size_t)(t - 1) * L + l) * dk;
        if (cudaMemcpyAsync(c->probes, pt, (size_t)dk, cudaMemcpyHostToDevice, c0->stream) != cudaSuccess) {
          rc = fail(COFEM_ECUDA, "probe upload");
          break;
        }
      } else {
        draw_stream_probes(c, t, K);  // c->stream is c0's stream here
      }
      const int64_t n = c->Dp * c->ldq;
      k_build_rhs<T><<<(int)std::min<int64_t>((n + 255) / 256, 8 * c->sm_count), 256, 0, c0->stream>>>(
          c->D, c->Dp, c->ldq, K, c->probes, 0, t, c->col_offset, c->aty, (T*)c->R, c->probe_store);
      c->launches++;
    }
    if (rc) break;
    cofem_cg_report rep;
    // one task IS the single-task solve (same kernels, same reduction order)
    rc = L == 1 ? pcg_device<T>(c0, betas[0], K + 1, 1, nullptr, cg, &rep)
                : pcg_multi<T>(cs, L, betas, K + 1, cg, &rep, agg, dptrs);
    if (steps) steps[t - 1] = rep.steps_taken;
    if (resid) resid[t - 1] = rep.final_relative_residual;
    if (rc == COFEM_EDIVERGED) {
      if (fail_it) *fail_it = t;
      if (fail_step) *fail_step = rep.steps_taken;
      rc = fail(COFEM_EDIVERGED, "non-finite residual at CG step " + std::to_string(rep.steps_taken) +
                                     " (EM iteration " + std::to_string(t) + ")");
      break;
    }
    if (rc) break;
    if (t == em->iterations && alpha) cudaMemcpyAsync(alpha, c0->alpha, c0->D * sizeof(double),
                                                       cudaMemcpyDeviceToHost, c0->stream);
    for (int l = 0; l < L; ++l) {
      cofem_ctx* c = cs[l];
      k_em_finish<T><<<(int)((c->D + 255) / 256), 256, 0, c0->stream>>>(
          c->D, c->ldq, K, betas[l], (const T*)c->X, c->probe_store, c->mu, c->s, c->alpha, c->minv, c->theta,
          em->theta_policy, 0, 0, em->floor_eps, em->clamp_max);
      c->launches++;
    }
    if (t < em->iterations) {
      k_multitask_alpha<<<(int)((c0->D + 255) / 256), 256, 0, c0->stream>>>(
          c0->D, L, dbeta, (const double* const*)aptrs, (const double* const*)(aptrs + L), aptrs + 2 * L,
          aptrs + 3 * L, (const double* const*)(aptrs + 4 * L), em->theta_policy, em->floor_eps, em->clamp_max);
      c0->launches++;
    }
    if (cudaGetLastError() != cudaSuccess) rc = fail(COFEM_ECUDA, "multitask kernels");
  }
  if (!rc) {
    cudaStreamSynchronize(c0->stream);
    for (int l = 0; l < L; ++l) {
      if (mus && mus[l]) cudaMemcpy(mus[l], cs[l]->mu, c0->D * sizeof(double), cudaMemcpyDeviceToHost);
      if (ss && ss[l]) cudaMemcpy(ss[l], cs[l]->s, c0->D * sizeof(double), cudaMemcpyDeviceToHost);
    }
  }
  cleanup();
  return rc;
}

// cg.solve_blocked with distinct systems (cg.py:201-234): block l is
// A_l X_l = B_l, A_l = beta_l Phi_l^T Phi_l + diag(alpha_l), with its own
// preconditioner; one lockstep PCG (pcg_multi) whose stopping rule aggregates
// the residual over all blocks.  Narrower blocks are zero-padded to the widest
// (a zero column freezes at its first step and never touches the aggregate).
template <typename T>
int pcg_solve_multi_impl(cofem_ctx** cs, int L, const double* betas, const double* const* alphas,
                         const double* const* minvs, const double* const* Bs, const int64_t* qs,
                         const cofem_cg_config* cg, double* const* Xs, cofem_cg_report* rep,
                         uint8_t* const* breakdowns) {
  cofem_ctx* c0 = cs[0];
  int64_t qmax = 1;
  for (int l = 0; l < L; ++l) qmax = std::max(qmax, qs[l]);
  const int ldq = ldq_for(qmax);
  if (ldq > 1024) return fail(COFEM_EINVAL, "at most 1024 right-hand sides per block");
  std::vector<cudaStream_t> saved(L);
  for (int l = 0; l < L; ++l) {
    cofem_ctx* c = cs[l];
    saved[l] = c->stream;
    CKR(ensure_ws(c, ldq));
    std::vector<double> a(c->Dp, 1.0), m(c->Dp, 0.0);
    std::copy(alphas[l], alphas[l] + c->D, a.begin());
    std::copy(minvs[l], minvs[l] + c->D, m.begin());
    CK(h2d_sync(c, c->alpha, a.data(), c->Dp * sizeof(double)));
    CK(h2d_sync(c, c->minv, m.data(), c->Dp * sizeof(double)));
    std::vector<double> b((size_t)c->D * qmax, 0.0);
    for (int64_t j = 0; j < c->D; ++j)
      for (int64_t k = 0; k < qs[l]; ++k) b[j * qmax + k] = Bs[l][j * qs[l] + k];
    CKR(upload_block<T>(c, b.data(), c->D, qmax, c->Dp, ldq, c->R));
  }
  CK(cudaDeviceSynchronize());
  for (int l = 0; l < L; ++l) cs[l]->stream = c0->stream;  // one stream for the lockstep
  double* agg = nullptr;
  double** dptrs = nullptr;
  int rc = 0;
  if (cudaMalloc(&agg, 2 * sizeof(double)) != cudaSuccess || cudaMalloc(&dptrs, 2 * L * sizeof(double*)) != cudaSuccess)
    rc = fail(COFEM_ENOMEM, "blocked solve tables");
  if (!rc) rc = pcg_multi<T>(cs, L, betas, (int)qmax, cg, rep, agg, dptrs);
  for (int l = 0; l < L; ++l) cs[l]->stream = saved[l];
  if (agg) cudaFree(agg);
  if (dptrs) cudaFree(dptrs);
  if (rc != 0 && rc != COFEM_EDIVERGED) return rc;
  int nb = 0;
  for (int l = 0; l < L; ++l) {
    cofem_ctx* c = cs[l];
    std::vector<double> x((size_t)c->D * qmax);
    CKR(download_block<T>(c, c->X, c->D, qmax, ldq, 0, x.data()));
    for (int64_t j = 0; j < c->D; ++j)
      for (int64_t k = 0; k < qs[l]; ++k) Xs[l][j * qs[l] + k] = x[j * qmax + k];
    std::vector<int> fz(ldq);
    CK(cudaMemcpy(fz.data(), c->frozen, ldq * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < qs[l]; ++k) {
      if (breakdowns && breakdowns[l]) breakdowns[l][k] = fz[k] ? 1 : 0;
      nb += fz[k] ? 1 : 0;
    }
  }
  rep->n_breakdown = nb;
  return rc;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int cofem_abi_version(void) { return COFEM_ABI_VERSION; }
const char* cofem_last_error(void) { return g_err.c_str(); }

int cofem_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return fail(COFEM_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *out = n;
  return 0;
}

int cofem_create(cofem_ctx** out, int device, int64_t n_rows, int64_t n_cols, int precision) {
  if (!out) return fail(COFEM_EINVAL, "null out");
  *out = nullptr;
  if (n_rows < 1 || n_cols < 1) return fail(COFEM_EINVAL, "operator dims must be positive");
  if (precision != COFEM_FP32 && precision != COFEM_FP64 && precision != COFEM_OZAKI && precision != COFEM_OZAKI24)
    return fail(COFEM_EINVAL, "precision must be FP32, FP64, OZAKI or OZAKI24");
  cofem_ctx* c = new cofem_ctx();
  c->device = device;
  c->prec = precision == COFEM_OZAKI24 ? COFEM_OZAKI : precision;
  c->npa = precision == COFEM_OZAKI24 ? 3 : 4;
  c->persistent_off = getenv("COFEM_NO_PERSISTENT") != nullptr;
  c->N = n_rows;
  c->D = n_cols;
  c->Np = round_up(n_rows, PAD);
  c->Dp = round_up(n_cols, PAD);
  c->global_cols = n_cols;
  auto bail = [&](int rc) {
    cofem_destroy(c);
    return rc;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(COFEM_ECUDA, "stream create failed"));
  if (cudaMalloc(&c->phi, (size_t)c->Np * c->Dp * sizeof(float)) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "dictionary allocation failed"));
  cudaMemsetAsync(c->phi, 0, (size_t)c->Np * c->Dp * sizeof(float), c->stream);
  double** dvecs[] = {&c->alpha, &c->minv, &c->theta, &c->colsq, &c->mu, &c->s, &c->aty};
  for (double** p : dvecs) {
    if (cudaMalloc(p, c->Dp * sizeof(double)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "vector allocation"));
    cudaMemsetAsync(*p, 0, c->Dp * sizeof(double), c->stream);
  }
  if (cudaMalloc(&c->tickets, 8 * sizeof(unsigned)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "tickets"));
  cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c->stream);
  if (cudaMalloc(&c->st, sizeof(Status)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "status"));
  if (cudaHostAlloc(&c->h_st, LAG * sizeof(Status), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->d_hst, c->h_st, 0) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "pinned status"));
  for (int i = 0; i < LAG; ++i) cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  cudaEventCreate(&c->t0);
  cudaEventCreate(&c->t1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, cudaGetErrorString(e)));
  cudaStreamSynchronize(c->stream);  // zero fills run on the context stream
  *out = c;
  return 0;
}

namespace {
// signed base-256 digits of round(x), host side (same decomposition as oz::digits4)
void host_digits(double x, int8_t* d, int n) {
  long long v = llrint(x);
  for (int a = n - 1; a >= 0; --a) {
    const int8_t lo = (int8_t)(v & 0xFF);
    d[a] = lo;
    v = (v - lo) >> 8;
  }
}
double host_pow2_ceil(double m) {
  int e;
  const double f = frexp(m, &e);
  return f == 0.5 ? ldexp(1.0, e - 1) : ldexp(1.0, e);
}
}  // namespace

int cofem_create_convolution(cofem_ctx** out, int device, int64_t dim, const double* taps, int64_t ntaps,
                             int precision) {
  if (!out || !taps) return fail(COFEM_EINVAL, "null argument");
  *out = nullptr;
  if (dim < 1 || ntaps < 1 || ntaps > dim) return fail(COFEM_EINVAL, "need 1 <= ntaps <= dim");
  const int npa = precision == COFEM_OZAKI24 ? 3 : 4;  // 24-bit taps: three band digit planes
  if (precision == COFEM_OZAKI24) precision = COFEM_OZAKI;
  if (precision != COFEM_OZAKI && precision != COFEM_FP64)
    return fail(COFEM_EINVAL, "convolution dictionaries run in OZAKI (int8 band) or FP64 (FFT) precision");
  if (precision == COFEM_FP64 && ntaps > CONV_FFT_MAX_TAPS)
    return fail(COFEM_EINVAL, "the FP64 (FFT) convolution path takes at most 512 taps");
  if (ntaps > oz::MAX_K_PER_ITEM - 2 * oz::BM) return fail(COFEM_EINVAL, "at most 32512 taps");
  double hmax = 0.0;
  for (int64_t m = 0; m < ntaps; ++m) {
    if (!std::isfinite(taps[m])) return fail(COFEM_EINVAL, "taps must be finite");
    hmax = std::max(hmax, std::fabs(taps[m]));
  }
  if (hmax == 0.0) return fail(COFEM_EINVAL, "all-zero filter");
  cofem_ctx* c = new cofem_ctx();
  c->kind = 1;
  c->device = device;
  c->prec = precision;
  c->npa = npa;
  c->N = c->D = dim;
  c->Np = c->Dp = round_up(dim, PAD);
  c->global_cols = dim;
  c->conv_L = (int)ntaps;
  c->conv_lpad = (int)round_up(ntaps - 1, oz::KT);
  c->taps.assign(taps, taps + ntaps);
  auto bail = [&](int rc) {
    cofem_destroy(c);
    return rc;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(COFEM_ECUDA, "stream create failed"));
  double** dvecs[] = {&c->alpha, &c->minv, &c->theta, &c->colsq, &c->mu, &c->s, &c->aty, &c->colscale, &c->hrows};
  for (double** p : dvecs) {
    if (cudaMalloc(p, c->Dp * sizeof(double)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "vector allocation"));
    cudaMemsetAsync(*p, 0, c->Dp * sizeof(double), c->stream);
  }
  if (cudaMalloc(&c->tickets, 8 * sizeof(unsigned)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "tickets"));
  cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c->stream);
  if (cudaMalloc(&c->st, sizeof(Status)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "status"));
  if (cudaHostAlloc(&c->h_st, LAG * sizeof(Status), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->d_hst, c->h_st, 0) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "pinned status"));
  for (int i = 0; i < LAG; ++i) cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  cudaEventCreate(&c->t0);
  cudaEventCreate(&c->t1);
  // column j of the lower-triangular Toeplitz matrix holds taps[0 : min(L, D - j)]
  {
    std::vector<double> csq(c->Dp, 0.0), cum(ntaps + 1, 0.0);
    for (int64_t m = 0; m < ntaps; ++m) cum[m + 1] = cum[m] + taps[m] * taps[m];
    for (int64_t j = 0; j < dim; ++j) csq[j] = cum[std::min<int64_t>(ntaps, dim - j)];
    h2d_sync(c, c->colsq, csq.data(), c->Dp * sizeof(double));
  }
  if (precision == COFEM_FP64) {
    // overlap-save spectra (1024 points, 1/1024 folded in) of h and of reversed h
    c->conv_fft = true;
    const int n = CONV_FFT_N;
    std::vector<double2> H(n), Hr(n), wN(n), w64(64);
    for (int k = 0; k < n; ++k) {
      double hr = 0, hi = 0, rr = 0, ri = 0;
      for (int64_t m = 0; m < ntaps; ++m) {
        const double ang = -2.0 * M_PI * (double)((k * m) % n) / n;
        hr += taps[m] * std::cos(ang);
        hi += taps[m] * std::sin(ang);
        const double tr = taps[ntaps - 1 - m];
        rr += tr * std::cos(ang);
        ri += tr * std::sin(ang);
      }
      H[k] = make_double2(hr / n, hi / n);
      Hr[k] = make_double2(rr / n, ri / n);
      wN[k] = make_double2(std::cos(2.0 * M_PI * k / n), -std::sin(2.0 * M_PI * k / n));
    }
    for (int j = 0; j < 64; ++j) w64[j] = make_double2(std::cos(2.0 * M_PI * j / 64), -std::sin(2.0 * M_PI * j / 64));
    if (cudaMalloc(&c->cf_H, n * sizeof(double2)) || cudaMalloc(&c->cf_Hr, n * sizeof(double2)) ||
        cudaMalloc(&c->dct_wN, n * sizeof(double2)) ||
        cudaMalloc(&c->colmax, 1024 * sizeof(unsigned long long)) != cudaSuccess)
      return bail(fail(COFEM_ENOMEM, "FFT tables"));
    h2d_sync(c, c->cf_H, H.data(), n * sizeof(double2));
    h2d_sync(c, c->cf_Hr, Hr.data(), n * sizeof(double2));
    h2d_sync(c, c->dct_wN, wN.data(), n * sizeof(double2));
    cudaMemcpyToSymbol(dctf::c_w64, w64.data(), 64 * sizeof(double2));
    e = cudaGetLastError();
    if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, cudaGetErrorString(e)));
    c->have_phi = true;
    cudaStreamSynchronize(c->stream);  // zero fills run on the context stream
  *out = c;
    return 0;
  }
  // operand buffers of the int8 path
  // operand planes with room for a neighbour's halo rows (time sharding):
  // lpad rows before P's planes, lpad rows after V's
  const size_t lpb = (size_t)4 * QCHUNK * c->conv_lpad;
  if (cudaMalloc(&c->pq_base, (size_t)4 * QCHUNK * c->Dp + lpb) != cudaSuccess ||
      cudaMalloc(&c->vq, (size_t)4 * QCHUNK * c->Np + lpb) != cudaSuccess ||
      cudaMalloc(&c->opscale, QCHUNK * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->colmax, 1024 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->vcolmax, QCHUNK * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->fz_max, 4 * 32 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "operand buffers"));
  c->conv_fused_off = getenv("COFEM_CONV_UNFUSED") != nullptr;
  cudaMemsetAsync(c->pq_base, 0, (size_t)4 * QCHUNK * c->Dp + lpb, c->stream);
  cudaMemsetAsync(c->vq, 0, (size_t)4 * QCHUNK * c->Np + lpb, c->stream);
  c->pq = c->pq_base + lpb;
  // band digit planes: lower band (Phi) and upper band (Phi^T), one scale 2^e >= max |h|;
  // npa planes of round(h / hs * 2^(8 npa - 2)) (the epilogue constant is the same for 3 and 4)
  const double hs = host_pow2_ceil(hmax);
  const double tsc = std::ldexp(1.0, 8 * npa - 2);
  const int nk = oz::BM + c->conv_lpad;
  std::vector<int8_t> bf((size_t)npa * oz::BM * nk, 0), ba((size_t)npa * oz::BM * nk, 0);
  for (int r = 0; r < oz::BM; ++r)
    for (int col = 0; col < nk; ++col) {
      const int mf = r + c->conv_lpad - col, ma = col - r;
      int8_t d[4];
      if (mf >= 0 && mf < ntaps) {
        host_digits(taps[mf] / hs * tsc, d, npa);
        for (int a = 0; a < npa; ++a) bf[((size_t)a * oz::BM + r) * nk + col] = d[a];
      }
      if (ma >= 0 && ma < ntaps) {
        host_digits(taps[ma] / hs * tsc, d, npa);
        for (int a = 0; a < npa; ++a) ba[((size_t)a * oz::BM + r) * nk + col] = d[a];
      }
    }
  if (cudaMalloc(&c->band_fwd, bf.size()) != cudaSuccess || cudaMalloc(&c->band_adj, ba.size()) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "band planes"));
  h2d_sync(c, c->band_fwd, bf.data(), bf.size());
  h2d_sync(c, c->band_adj, ba.data(), ba.size());
  int rc = encode_u8_3d(&c->map_band_fwd, c->band_fwd, nk, oz::BM, npa, oz::KT, oz::BM, npa);
  if (!rc) rc = encode_u8_3d(&c->map_band_adj, c->band_adj, nk, oz::BM, npa, oz::KT, oz::BM, npa);
  if (rc) return bail(rc);
  // scales: output rows carry hs; operands are not pre-scaled (ones)
  std::vector<double> hv(c->Dp, hs), ones(c->Dp, 1.0);
  h2d_sync(c, c->hrows, hv.data(), c->Dp * sizeof(double));
  h2d_sync(c, c->colscale, ones.data(), c->Dp * sizeof(double));
  e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, cudaGetErrorString(e)));
  c->have_phi = true;
  c->oz_ready = true;
  cudaStreamSynchronize(c->stream);  // zero fills run on the context stream
  *out = c;
  return 0;
}

int cofem_create_dct1(cofem_ctx** out, int device, int64_t dim, const int64_t* mask, int64_t nmask, int precision) {
  if (!out || !mask) return fail(COFEM_EINVAL, "null argument");
  *out = nullptr;
  if (dim < 2 || dim > ((int64_t)1 << 30)) return fail(COFEM_EINVAL, "need 2 <= dim <= 2^30");
  if (nmask < 1 || nmask > dim) return fail(COFEM_EINVAL, "need 1 <= mask size <= dim");
  if (precision == COFEM_OZAKI24 || precision == COFEM_OZAKI) precision = COFEM_FP64;
  if (precision != COFEM_FP64) return fail(COFEM_EINVAL, "1-D DCT dictionaries run in FP64 (cuFFT double complex)");
  std::vector<uint8_t> grid((size_t)dim, 0);
  for (int64_t m = 0; m < nmask; ++m) {
    if (mask[m] < 0 || mask[m] >= dim) return fail(COFEM_EINVAL, "mask indices must lie in [0, dim)");
    if (grid[mask[m]]) return fail(COFEM_EINVAL, "mask indices must be distinct");
    grid[mask[m]] = 1;
  }
  CKR(cufft_load());
  cofem_ctx* c = new cofem_ctx();
  c->kind = 3;
  c->device = device;
  c->prec = COFEM_FP64;
  c->N = nmask;
  c->D = dim;
  c->Np = round_up(nmask, PAD);
  c->Dp = round_up(dim, PAD);
  c->global_cols = dim;
  auto bail = [&](int rc) {
    cofem_destroy(c);
    return rc;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(COFEM_ECUDA, "stream create failed"));
  double** dvecs[] = {&c->alpha, &c->minv, &c->theta, &c->colsq, &c->mu, &c->s, &c->aty};
  for (double** p : dvecs) {
    if (cudaMalloc(p, c->Dp * sizeof(double)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "vector allocation"));
    cudaMemsetAsync(*p, 0, c->Dp * sizeof(double), c->stream);
  }
  if (cudaMalloc(&c->tickets, 8 * sizeof(unsigned)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "tickets"));
  cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c->stream);
  if (cudaMalloc(&c->st, sizeof(Status)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "status"));
  if (cudaHostAlloc(&c->h_st, LAG * sizeof(Status), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->d_hst, c->h_st, 0) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "pinned status"));
  for (int i = 0; i < LAG; ++i) cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  cudaEventCreate(&c->t0);
  cudaEventCreate(&c->t1);
  if (cudaMalloc(&c->colmax, 1024 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "colmax"));
  // the mask sorted (row order of Phi) and in Makhoul order: mv[m] = grid[sigma(m)]
  std::vector<int64_t> sorted(mask, mask + nmask);
  std::sort(sorted.begin(), sorted.end());
  std::vector<uint8_t> mv((size_t)dim);
  for (int64_t m = 0; m < dim; ++m) mv[m] = grid[m < (dim + 1) / 2 ? 2 * m : 2 * (dim - 1 - m) + 1];
  if (cudaMalloc(&c->dct_mask, nmask * sizeof(int64_t)) || cudaMalloc(&c->dct1_mv, (size_t)dim))
    return bail(fail(COFEM_ENOMEM, "DCT tables"));
  h2d_sync(c, c->dct_mask, sorted.data(), nmask * sizeof(int64_t));
  h2d_sync(c, c->dct1_mv, mv.data(), (size_t)dim);
  e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, cudaGetErrorString(e)));
  c->have_phi = true;
  c->oz_ready = true;
  cudaStreamSynchronize(c->stream);
  *out = c;
  return 0;
}

int cofem_create_dct2(cofem_ctx** out, int device, int64_t n, const int64_t* mask, int64_t nmask, int precision) {
  if (!out || !mask) return fail(COFEM_EINVAL, "null argument");
  *out = nullptr;
  if (n < 64 || n > 1024 || (n & (n - 1)) != 0) return fail(COFEM_EINVAL, "image side must be a power of two in [64, 1024]");
  if (nmask < 1 || nmask > n * n) return fail(COFEM_EINVAL, "need 1 <= mask size <= n^2");
  if (precision == COFEM_OZAKI24) precision = COFEM_OZAKI;
  if (precision != COFEM_OZAKI && precision != COFEM_FP64)
    return fail(COFEM_EINVAL, "2-D DCT dictionaries run in FP64 (fused FFT passes; OZAKI is accepted as an alias)");
  std::vector<uint8_t> grid((size_t)n * n, 0);
  for (int64_t m = 0; m < nmask; ++m) {
    if (mask[m] < 0 || mask[m] >= n * n) return fail(COFEM_EINVAL, "mask indices must lie in [0, n^2)");
    if (grid[mask[m]]) return fail(COFEM_EINVAL, "mask indices must be distinct");
    grid[mask[m]] = 1;
  }
  cofem_ctx* c = new cofem_ctx();
  c->kind = 2;
  c->device = device;
  c->prec = COFEM_FP64;  // float64 FFT passes whatever the requested mode
  c->dct_n = (int)n;
  c->N = nmask;
  c->D = n * n;
  c->Np = round_up(nmask, PAD);
  c->Dp = round_up(c->D, PAD);
  c->global_cols = c->D;
  auto bail = [&](int rc) {
    cofem_destroy(c);
    return rc;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(COFEM_ECUDA, "stream create failed"));
  double** dvecs[] = {&c->alpha, &c->minv, &c->theta, &c->colsq, &c->mu, &c->s, &c->aty};
  for (double** p : dvecs) {
    if (cudaMalloc(p, c->Dp * sizeof(double)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "vector allocation"));
    cudaMemsetAsync(*p, 0, c->Dp * sizeof(double), c->stream);
  }
  if (cudaMalloc(&c->tickets, 8 * sizeof(unsigned)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "tickets"));
  cudaMemsetAsync(c->tickets, 0, 8 * sizeof(unsigned), c->stream);
  if (cudaMalloc(&c->st, sizeof(Status)) != cudaSuccess) return bail(fail(COFEM_ENOMEM, "status"));
  if (cudaHostAlloc(&c->h_st, LAG * sizeof(Status), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->d_hst, c->h_st, 0) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "pinned status"));
  for (int i = 0; i < LAG; ++i) cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  cudaEventCreate(&c->t0);
  cudaEventCreate(&c->t1);
  if (cudaMalloc(&c->colmax, 1024 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(COFEM_ENOMEM, "colmax"));
  // FFT tables: w_n^j = e^{-2 pi i j / n}, Makhoul twiddles e^{-i pi k / 2n},
  // orthonormal scales c_k; the register DFTs' e^{-2 pi i j / 64} in __constant__
  std::vector<double2> wN(n), tw(n), w64(64);
  std::vector<double> cn(n);
  for (int64_t j = 0; j < n; ++j) {
    wN[j] = make_double2(std::cos(2.0 * M_PI * j / n), -std::sin(2.0 * M_PI * j / n));
    // the Makhoul twiddles carry the pair steps' common scale c_k / 2 = 1 / (c_k n) = 1 / sqrt(2n)
    tw[j] = make_double2(std::cos(M_PI * j / (2.0 * n)) / std::sqrt(2.0 * n), -std::sin(M_PI * j / (2.0 * n)) / std::sqrt(2.0 * n));
    cn[j] = j == 0 ? std::sqrt(1.0 / n) : std::sqrt(2.0 / n);
  }
  for (int j = 0; j < 64; ++j) w64[j] = make_double2(std::cos(2.0 * M_PI * j / 64), -std::sin(2.0 * M_PI * j / 64));
  if (cudaMalloc(&c->dct_wN, n * sizeof(double2)) || cudaMalloc(&c->dct_tw, n * sizeof(double2)) ||
      cudaMalloc(&c->dct_cn, n * sizeof(double)) || cudaMalloc(&c->dct_mask, nmask * sizeof(int64_t)) ||
      cudaMalloc(&c->dct_grid, grid.size()) || cudaMalloc(&c->dct_gridT, grid.size()))
    return bail(fail(COFEM_ENOMEM, "DCT tables"));
  h2d_sync(c, c->dct_wN, wN.data(), n * sizeof(double2));
  h2d_sync(c, c->dct_tw, tw.data(), n * sizeof(double2));
  h2d_sync(c, c->dct_cn, cn.data(), n * sizeof(double));
  cudaMemcpyToSymbol(dctf::c_w64, w64.data(), 64 * sizeof(double2));
  std::vector<int64_t> sorted(mask, mask + nmask);
  std::sort(sorted.begin(), sorted.end());
  h2d_sync(c, c->dct_mask, sorted.data(), nmask * sizeof(int64_t));
  h2d_sync(c, c->dct_grid, grid.data(), grid.size());
  std::vector<uint8_t> gridT(grid.size());
  for (int64_t k = 0; k < n; ++k)
    for (int64_t l = 0; l < n; ++l) gridT[l * n + k] = grid[k * n + l];
  h2d_sync(c, c->dct_gridT, gridT.data(), gridT.size());
  {
    const int n1 = n == 64 ? 8 : n == 128 ? 8 : n == 256 ? 16 : n == 512 ? 16 : 32, n2 = (int)n / n1;
    std::vector<double2> wT(n);
    for (int k2 = 0; k2 < n2; ++k2)
      for (int lt = 0; lt < n1; ++lt) wT[k2 * n1 + lt] = wN[lt * k2];
    if (cudaMalloc(&c->dct_wT, n * sizeof(double2))) return bail(fail(COFEM_ENOMEM, "DCT tables"));
    h2d_sync(c, c->dct_wT, wT.data(), n * sizeof(double2));
  }
  if (cudaMalloc(&c->dct_fscal, 4 * PSQ * sizeof(double)) ||
      cudaMalloc(&c->dct_partials, (size_t)16 * c->sm_count * dctf::VV_MAXQ * sizeof(double)) ||
      cudaMalloc(&c->dct_partials4, (size_t)3 * c->sm_count * 4 * PSQ * sizeof(double)))
    return bail(fail(COFEM_ENOMEM, "DCT step scalars"));
  cudaMemsetAsync(c->dct_fscal, 0, 4 * PSQ * sizeof(double), c->stream);
  if (n == 1024 && getenv("COFEM_DCT_WARP")) {  // tables of the warp-per-FFT passes (dct1024.cuh)
    std::vector<double2> twF(1024);
    for (int k2 = 0; k2 < 32; ++k2)
      for (int lt = 0; lt < 32; ++lt) twF[k2 * 32 + lt] = wN[lt * k2];
    std::vector<uint8_t> pm((size_t)n * 512);
    for (int64_t o = 0; o < n; ++o)
      for (int lt = 0; lt < 32; ++lt)
        for (int k1 = 0; k1 < 16; ++k1) {
          const int k = lt + 32 * k1;
          uint8_t b = gridT[o * n + k];
          if (k > 0) b |= gridT[o * n + (n - k)] << 1;
          if (k == 0) b |= gridT[o * n + 512] << 2;
          pm[(o * 32 + lt) * 16 + k1] = b;
        }
    if (cudaMalloc(&c->dct_twF, 1024 * sizeof(double2)) || cudaMalloc(&c->dct_pm, pm.size()))
      return bail(fail(COFEM_ENOMEM, "DCT tables"));
    h2d_sync(c, c->dct_twF, twF.data(), 1024 * sizeof(double2));
    h2d_sync(c, c->dct_pm, pm.data(), pm.size());
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(COFEM_ECUDA, cudaGetErrorString(e)));
  c->have_phi = true;
  c->oz_ready = true;
  cudaStreamSynchronize(c->stream);  // zero fills run on the context stream
  *out = c;
  return 0;
}

int cofem_destroy(cofem_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_ws(c);
  void* ptrs[] = {c->gbar, c->ptimes, c->phi, c->phi64, c->alpha, c->minv, c->theta, c->colsq, c->mu, c->s, c->aty, c->ybuf,
                  c->probes, c->probe_store, c->groups, c->tickets, c->st, c->phiq, c->phiqT, c->rowscale, c->colscale,
                  c->pq_base ? c->pq_base : c->pq, c->vq, c->opscale, c->colmax, c->vcolmax, c->band_fwd, c->band_adj, c->hrows,
                  c->dct_mask, c->dct_grid, c->dct_gridT, c->bufA, c->bufB, c->dct_wN, c->dct_tw, c->dct_cn,
                  c->cf_H, c->cf_Hr, c->lg_tmp, c->fz_max, c->dct1_mv, c->dct_twF, c->dct_pm, c->dct_wT, c->dct_fscal, c->dct_partials, c->dct_partials4};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->h_st) cudaFreeHost(c->h_st);
  for (int i = 0; i < LAG; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  for (cudaEvent_t e : c->evpool) cudaEventDestroy(e);
  if (c->fft_plan_hc && g_cufft.ok) g_cufft.destroy(c->fft_plan);
  if (c->comm && g_nccl.ok) g_nccl.commDestroy(c->comm);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}



int cofem_set_dictionary(cofem_ctx* c, const float* phi, int64_t ld, int on_device) {
  CKR(check_ctx(c, false));
  if (c->kind != 0) return fail(COFEM_EINVAL, "not a dense dictionary context");
  if (!phi || ld < c->D) return fail(COFEM_EINVAL, "dictionary pointer / leading dimension");
  if (on_device)
    CK(cudaMemcpy2DAsync(c->phi, c->Dp * sizeof(float), phi, ld * sizeof(float), c->D * sizeof(float), c->N,
                         cudaMemcpyDeviceToDevice, c->stream));
  else
    CKR(upload_rows(c, c->phi, c->Dp * sizeof(float), phi, ld * sizeof(float), c->D * sizeof(float), c->N));
  CK(cudaStreamSynchronize(c->stream));
  if (c->phi64) {  // a float32 dictionary replaces an earlier float64 one
    cudaFree(c->phi64);
    c->phi64 = nullptr;
  }
  c->have_phi = true;
  c->oz_ready = false;
  return 0;
}

namespace {
__global__ void k_round_f32(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = (float)src[e];
}
}  // namespace

int cofem_set_dictionary_f64(cofem_ctx* c, const double* phi, int64_t ld) {
  CKR(check_ctx(c, false));
  if (c->kind != 0) return fail(COFEM_EINVAL, "not a dense dictionary context");
  if (!phi || ld < c->D) return fail(COFEM_EINVAL, "dictionary pointer / leading dimension");
  double* tmp = nullptr;
  const size_t bytes = (size_t)c->Np * c->Dp * sizeof(double);
  CK(cudaMalloc(&tmp, bytes));
  CK(cudaMemsetAsync(tmp, 0, bytes, c->stream));
  int rc = 0;
  rc = upload_rows(c, tmp, c->Dp * sizeof(double), phi, ld * sizeof(double), c->D * sizeof(double), c->N);
  if (!rc) {
    // the float32 copy serves cofem_get_dictionary (and the fp32 mode)
    k_round_f32<<<16 * c->sm_count, 256, 0, c->stream>>>(tmp, c->phi, (int64_t)c->Np * c->Dp);
    c->launches++;
    c->oz_ready = false;
    if (c->prec == COFEM_OZAKI) rc = ensure_oz(c, tmp);  // planes from the exact float64 values
  }
  cudaStreamSynchronize(c->stream);
  if (c->phi64) cudaFree(c->phi64);
  c->phi64 = nullptr;
  if (!rc && c->prec == COFEM_FP64) c->phi64 = tmp;  // fp64 mode multiplies the exact float64 entries
  else cudaFree(tmp);
  if (!rc) c->have_phi = true;
  return rc;
}

int cofem_set_shard(cofem_ctx* c, int64_t col_offset, int64_t global_cols) {
  if (!c) return fail(COFEM_EINVAL, "null context");
  if (col_offset < 0 || col_offset + c->D > global_cols || col_offset % 4 != 0)
    return fail(COFEM_EINVAL, "shard must be 4-aligned and inside the global columns");
  if ((c->kind == 2 || c->kind == 3) && (col_offset != 0 || global_cols != c->D))
    return fail(COFEM_EINVAL, "2-D DCT dictionaries are not sharded");
  if (c->kind == 1) {
    // time shard [t0, t0 + D) of a length-global_cols sequence: boundaries on
    // PAD-row multiples, and a shard followed by another one holds at least
    // the halo (the neighbours exchange only lpad rows)
    if (col_offset % PAD != 0) return fail(COFEM_EINVAL, "convolution shards start on 256-sample boundaries");
    if (col_offset + c->D < global_cols && (c->D % PAD != 0 || c->D < c->conv_lpad))
      return fail(COFEM_EINVAL, "inner convolution shards need a multiple of 256 samples and >= the filter halo");
    if (c->conv_fft && global_cols != c->D) return fail(COFEM_EINVAL, "the FP64 FFT convolution path is not sharded");
    // column j of the global Toeplitz matrix holds taps[0 : min(L, global - j)]
    const int64_t L = (int64_t)c->taps.size();
    std::vector<double> csq(c->Dp, 0.0), cum(L + 1, 0.0);
    for (int64_t m = 0; m < L; ++m) cum[m + 1] = cum[m] + c->taps[m] * c->taps[m];
    for (int64_t j = 0; j < c->D; ++j) csq[j] = cum[std::min<int64_t>(L, global_cols - col_offset - j)];
    CKR(set_dev(c));
    CK(h2d_sync(c, c->colsq, csq.data(), c->Dp * sizeof(double)));
  }
  c->col_offset = col_offset;
  c->global_cols = global_cols;
  return 0;
}

namespace {
// shared by cofem_set_comm / cofem_set_group: what may be sharded, and how
int attach_ranks(cofem_ctx* c, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(COFEM_EINVAL, "bad rank / nranks");
  if (nranks > 1) {
    if (c->kind == 2 || c->kind == 3) return fail(COFEM_EINVAL, "DCT dictionaries run on one GPU (not sharded)");
    if (c->kind == 1 && c->conv_fft) return fail(COFEM_EINVAL, "the FP64 FFT convolution path runs on one GPU");
    if (c->kind == 1 && c->col_offset + c->D < c->global_cols && rank == nranks - 1)
      return fail(COFEM_EINVAL, "the last rank must hold the end of the sequence");
  }
  c->nranks = nranks;
  c->rank = rank;
  // dense shards share the row scales of the whole dictionary: rebuild the
  // digit planes (collectively, on first use) if they were made before joining
  if (c->kind == 0 && nranks > 1) c->oz_ready = false;
  // operand maps depend on the neighbours (halo extents): re-encode on next use
  for (int i = 0; i < 5; ++i) c->map_p_ok[i] = c->map_v_ok[i] = false;
  return 0;
}
}  // namespace

int cofem_group_create(cofem_group** out, int nranks) {
  if (!out) return fail(COFEM_EINVAL, "null argument");
  *out = nullptr;
  if (nranks < 1 || nranks > GROUP_MAX) return fail(COFEM_EINVAL, "a shard group holds 1..8 ranks");
  cofem_group* g = new cofem_group();
  g->n = nranks;
  g->bufs.assign(nranks, nullptr);
  g->ready.assign(nranks, nullptr);
  g->done.assign(nranks, nullptr);
  *out = g;
  return 0;
}

int cofem_group_destroy(cofem_group* g) {
  if (!g) return 0;
  for (cudaEvent_t e : g->ready)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : g->done)
    if (e) cudaEventDestroy(e);
  delete g;
  return 0;
}

int cofem_group_abort(cofem_group* g) {
  group_break(g);
  return 0;
}

int cofem_set_group(cofem_ctx* c, cofem_group* g, int rank) {
  CKR(check_ctx(c, false));
  if (!g) return fail(COFEM_EINVAL, "null group");
  if (c->comm) return fail(COFEM_ESTATE, "context already joined an NCCL communicator");
  if (rank < 0 || rank >= g->n) return fail(COFEM_EINVAL, "bad rank");
  if (g->ready[rank]) return fail(COFEM_ESTATE, "rank already attached to this group");
  CKR(attach_ranks(c, g->n, rank));
  CKR(set_dev(c));
  // peers on other devices are read directly: enable peer access both ways
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  for (int d = 0; d < ndev; ++d)
    if (d != c->device) {
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, c->device, d);
      if (ok) cudaDeviceEnablePeerAccess(d, 0);
    }
  cudaGetLastError();  // (already-enabled peers)
  CK(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming));
  c->lgroup = g;
  return 0;
}

int cofem_generate_gaussian_dictionary(cofem_ctx* c, uint64_t seed, double scale) {
  CKR(check_ctx(c, false));
  if (c->kind != 0) return fail(COFEM_EINVAL, "not a dense dictionary context");
  const int64_t total = c->N * ((c->D + 3) / 4);
  const int gs = (int)std::min<int64_t>((total + 255) / 256, 64 * c->sm_count);
  k_gen_gaussian<<<gs, 256, 0, c->stream>>>(c->phi, c->Dp, c->N, c->D, c->col_offset, seed, scale);
  if (c->phi64) {
    cudaFree(c->phi64);
    c->phi64 = nullptr;
  }
  c->launches++;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  c->have_phi = true;
  c->oz_ready = false;
  return 0;
}

int cofem_get_dictionary(cofem_ctx* c, float* out) {
  CKR(check_ctx(c));
  if (c->kind != 0) return fail(COFEM_EINVAL, "not a dense dictionary context");
  CK(cudaMemcpy2D(out, c->D * sizeof(float), c->phi, c->Dp * sizeof(float), c->D * sizeof(float), c->N,
                  cudaMemcpyDeviceToHost));
  return 0;
}

int cofem_nccl_get_unique_id(void* out128) {
  CKR(nccl_load());
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) return fail(COFEM_ENCCL, "ncclGetUniqueId failed");
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int cofem_set_comm(cofem_ctx* c, const void* uid, int nranks, int rank) {
  CKR(check_ctx(c, false));
  if (c->lgroup) return fail(COFEM_ESTATE, "context already joined a shard group");
  CKR(attach_ranks(c, nranks, rank));
  CKR(nccl_load());
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclResult_t r = g_nccl.commInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) return fail(COFEM_ENCCL, std::string("ncclCommInitRank: ") + (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
  c->nranks = nranks;
  c->rank = rank;
  return 0;
}

#define DISPATCH(c, fn, ...) ((c)->prec == COFEM_FP32 ? fn<float>(__VA_ARGS__) : fn<double>(__VA_ARGS__))

namespace {
// a rank that fails outside an exchange releases the group's other ranks
int grouped(cofem_ctx* c, int rc) {
  if (rc && rc != COFEM_EDIVERGED && c->lgroup) group_break(c->lgroup);
  return rc;
}
}  // namespace

int cofem_apply(cofem_ctx* c, const double* V, int64_t q, double* out) {
  CKR(check_ctx(c));
  if (q < 1) return fail(COFEM_EINVAL, "q must be >= 1");
  return grouped(c, DISPATCH(c, apply_impl, c, V, q, out));
}

int cofem_apply_adjoint(cofem_ctx* c, const double* U, int64_t q, double* out) {
  CKR(check_ctx(c));
  if (q < 1) return fail(COFEM_EINVAL, "q must be >= 1");
  return grouped(c, DISPATCH(c, adjoint_impl, c, U, q, out));
}

int cofem_system_apply(cofem_ctx* c, double beta, const double* alpha, const double* V, int64_t q, double* out) {
  CKR(check_ctx(c));
  if (q < 1) return fail(COFEM_EINVAL, "q must be >= 1");
  if (!(beta > 0)) return fail(COFEM_EINVAL, "beta must be positive");
  return grouped(c, DISPATCH(c, system_apply_impl, c, beta, alpha, V, q, out));
}

int cofem_column_sq_norms(cofem_ctx* c, double* out) {
  CKR(check_ctx(c));
  if (c->kind == 1) {
    CK(cudaMemcpy(out, c->colsq, c->D * sizeof(double), cudaMemcpyDeviceToHost));
    return 0;
  }
  if (c->kind == 2 || c->kind == 3)
    return fail(COFEM_EINVAL, "DCT column norms are computed by the host (pass a custom theta)");
  CKR(dense_colsq(c));
  CK(cudaMemcpyAsync(out, c->colsq, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

}  // extern "C"

namespace {
template <typename T>
int pcg_solve_impl(cofem_ctx* c, double beta, const double* alpha, const double* minv, int32_t ngroups,
                   const int32_t* group_of_col, const double* B, int64_t q, const cofem_cg_config* cg, double* X,
                   cofem_cg_report* rep, uint8_t* breakdown) {
  const int ldq = ldq_for(q);
  if (ldq > 1024) return fail(COFEM_EINVAL, "at most 1024 right-hand sides per solve");
  CKR(ensure_ws(c, ldq));
  std::vector<double> a(c->Dp, 0.0);
  std::copy(alpha, alpha + c->D, a.begin());
  CK(h2d_sync(c, c->alpha, a.data(), c->Dp * sizeof(double)));
  // minv: D x ngroups (groups > 1 stored in a dedicated buffer)
  double* minv_dev = c->minv;
  double* minv_tmp = nullptr;
  if (ngroups > 1) {
    CK(cudaMalloc(&minv_tmp, (size_t)c->Dp * ngroups * sizeof(double)));
    minv_dev = minv_tmp;
  }
  std::vector<double> m((size_t)c->Dp * ngroups, 0.0);
  std::copy(minv, minv + (size_t)c->D * ngroups, m.begin());
  CK(h2d_sync(c, minv_dev, m.data(), m.size() * sizeof(double)));
  int* gdev = nullptr;
  if (ngroups > 1) {
    std::vector<int> g(ldq, 0);
    for (int64_t k = 0; k < q; ++k) g[k] = group_of_col[k];
    CKR(ensure_groups(c, ldq));
    CK(h2d_sync(c, c->groups, g.data(), ldq * sizeof(int)));
    gdev = c->groups;
  }
  CKR(upload_block<T>(c, B, c->D, q, c->Dp, ldq, c->R));
  // pcg_device reads c->minv: temporarily swap in the grouped one
  double* saved = c->minv;
  c->minv = minv_dev;
  int rc = pcg_device<T>(c, beta, (int)q, ngroups, gdev, cg, rep);
  c->minv = saved;
  if (minv_tmp) cudaFree(minv_tmp);
  if (rc != 0 && rc != COFEM_EDIVERGED) return rc;
  CKR(download_block<T>(c, c->X, c->D, q, ldq, 0, X));
  if (breakdown) {
    std::vector<int> fz(ldq);
    CK(cudaMemcpy(fz.data(), c->frozen, ldq * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < q; ++k) breakdown[k] = fz[k] ? 1 : 0;
  }
  return rc;
}
}  // namespace

extern "C" {

int cofem_pcg_solve(cofem_ctx* c, double beta, const double* alpha, const double* minv, int32_t n_groups,
                    const int32_t* group_of_col, const double* B, int64_t q, const cofem_cg_config* cg, double* X,
                    cofem_cg_report* rep, uint8_t* breakdown) {
  CKR(check_ctx(c));
  if (!alpha || !minv || !B || !X || !cg || !rep || q < 1) return fail(COFEM_EINVAL, "null argument");
  if (cg->max_steps < 1 || !(cg->tolerance > 0)) return fail(COFEM_EINVAL, "bad CG config");
  if (n_groups < 1 || (n_groups > 1 && !group_of_col)) return fail(COFEM_EINVAL, "bad groups");
  return grouped(c, DISPATCH(c, pcg_solve_impl, c, beta, alpha, minv, n_groups, group_of_col, B, q, cg, X, rep, breakdown));
}

int cofem_run(cofem_ctx* c, const double* y, double beta, const cofem_em_config* em, const cofem_cg_config* cg,
              const double* theta, const int8_t* probes, uint64_t dseed, double* alpha, double* mu, double* s,
              int32_t* cg_steps, double* cg_residuals, int32_t* failed_iteration, int32_t* failed_step) {
  CKR(check_ctx(c));
  if (!y || !em || !cg) return fail(COFEM_EINVAL, "null argument");
  if (em->iterations < 1 || em->probes < 1) return fail(COFEM_EINVAL, "iterations and probes must be >= 1");
  if (em->probes + 1 > 1024) return fail(COFEM_EINVAL, "too many probes");
  if (cg->max_steps < 1 || !(cg->tolerance > 0)) return fail(COFEM_EINVAL, "bad CG config");
  if (!(beta > 0) || !std::isfinite(beta)) return fail(COFEM_EINVAL, "beta must be positive and finite");
  return grouped(c, DISPATCH(c, run_impl, c, y, beta, em, cg, theta, probes, dseed, alpha, mu, s, cg_steps,
                             cg_residuals, failed_iteration, failed_step));
}

int cofem_run_multitask(cofem_ctx* const* ctxs, int n_tasks, const double* const* ys, const double* betas,
                        const cofem_em_config* em, const cofem_cg_config* cg, const double* theta,
                        const int8_t* probes, double* alpha, double* const* mus, double* const* ss,
                        int32_t* cg_steps, double* cg_residuals, int32_t* failed_iteration, int32_t* failed_step) {
  if (!ctxs || n_tasks < 1 || !ys || !betas || !em || !cg) return fail(COFEM_EINVAL, "null argument");
  cofem_ctx* c0 = ctxs[0];
  CKR(check_ctx(c0));
  if (em->variant != COFEM_STANDARD) return fail(COFEM_EINVAL, "multi-task loop supports the standard variant only");
  if (em->iterations < 1 || em->probes < 1 || em->probes + 1 > 1024) return fail(COFEM_EINVAL, "bad EM config");
  if (cg->max_steps < 1 || !(cg->tolerance > 0)) return fail(COFEM_EINVAL, "bad CG config");
  for (int l = 0; l < n_tasks; ++l) {
    cofem_ctx* c = ctxs[l];
    if (!(betas[l] > 0) || !std::isfinite(betas[l])) return fail(COFEM_EINVAL, "beta must be positive and finite");
    CKR(check_ctx(c));
    if (c->D != c0->D || c->prec != c0->prec || c->device != c0->device || c->nranks > 1)
      return fail(COFEM_EINVAL, "tasks must share D, precision and device (single GPU)");
    for (int m = 0; m < l; ++m)
      if (ctxs[m] == c) return fail(COFEM_EINVAL, "each task needs its own context");
    if (!probes && !c->pcg_stream) return fail(COFEM_EINVAL, "no probes: pass host signs or set a probe stream");
  }
  std::vector<cofem_ctx*> cs(ctxs, ctxs + n_tasks);
  return DISPATCH(c0, run_multi_impl, cs.data(), n_tasks, ys, betas, em, cg, theta, probes, alpha, mus, ss,
                  cg_steps, cg_residuals, failed_iteration, failed_step);
}

int cofem_last_run_report(cofem_ctx* c, int32_t iterations, double* wall_times, double* solution,
                          uint8_t* breakdown, cofem_cg_report* rep) {
  CKR(check_ctx(c));
  if (c->run_K < 1) return fail(COFEM_ESTATE, "no completed cofem_run on this context");
  if (wall_times) {
    if (iterations != (int32_t)c->run_wall.size()) return fail(COFEM_EINVAL, "iterations != the last run's T");
    std::copy(c->run_wall.begin(), c->run_wall.end(), wall_times);
  }
  const int q = c->run_K + 1;
  if (solution) CKR(DISPATCH(c, download_block, c, c->X, c->D, q, c->ldq, 0, solution));
  if (breakdown) {
    std::vector<int> fz(c->ldq);
    CK(cudaMemcpy(fz.data(), c->frozen, c->ldq * sizeof(int), cudaMemcpyDeviceToHost));
    for (int k = 0; k < q; ++k) breakdown[k] = fz[k] ? 1 : 0;
  }
  if (rep) *rep = c->run_rep;
  return 0;
}

int cofem_pcg_solve_multi(cofem_ctx* const* ctxs, int n_blocks, const double* betas, const double* const* alphas,
                          const double* const* minvs, const double* const* Bs, const int64_t* qs,
                          const cofem_cg_config* cg, double* const* Xs, cofem_cg_report* rep,
                          uint8_t* const* breakdowns) {
  if (!ctxs || n_blocks < 1 || !betas || !alphas || !minvs || !Bs || !qs || !cg || !Xs || !rep)
    return fail(COFEM_EINVAL, "null argument");
  if (cg->max_steps < 1 || !(cg->tolerance > 0)) return fail(COFEM_EINVAL, "bad CG config");
  cofem_ctx* c0 = ctxs[0];
  CKR(check_ctx(c0));
  for (int l = 0; l < n_blocks; ++l) {
    cofem_ctx* c = ctxs[l];
    CKR(check_ctx(c));
    if (!alphas[l] || !minvs[l] || !Bs[l] || !Xs[l] || qs[l] < 1) return fail(COFEM_EINVAL, "null block argument");
    if (!(betas[l] > 0) || !std::isfinite(betas[l])) return fail(COFEM_EINVAL, "beta must be positive and finite");
    if (c->D != c0->D || c->prec != c0->prec || c->device != c0->device || c->nranks > 1)
      return fail(COFEM_EINVAL, "blocks must share D, precision and device (single GPU)");
    for (int m = 0; m < l; ++m)
      if (ctxs[m] == c) return fail(COFEM_EINVAL, "each block needs its own context");
  }
  std::vector<cofem_ctx*> cs(ctxs, ctxs + n_blocks);
  CKR(set_dev(c0));
  return DISPATCH(c0, pcg_solve_multi_impl, cs.data(), n_blocks, betas, alphas, minvs, Bs, qs, cg, Xs, rep,
                  breakdowns);
}

int cofem_set_probe_stream_ex(cofem_ctx* c, const uint64_t* state, const uint64_t* inc, uint64_t first_half,
                              uint64_t halves_per_iteration) {
  CKR(check_ctx(c));
  if (!state || !inc) {
    c->pcg_stream = false;
    return 0;
  }
  if (!(inc[1] & 1)) return fail(COFEM_EINVAL, "PCG64 increment must be odd");
  c->pcg_stream = true;
  c->pcg_state[0] = state[0];
  c->pcg_state[1] = state[1];
  c->pcg_inc[0] = inc[0];
  c->pcg_inc[1] = inc[1];
  c->pcg_first = first_half;
  c->pcg_stride = halves_per_iteration;
  return 0;
}

int cofem_set_probe_stream(cofem_ctx* c, const uint64_t* state, const uint64_t* inc) {
  return cofem_set_probe_stream_ex(c, state, inc, 0, 0);
}

int cofem_pcg64_rademacher(int device, const uint64_t* state, const uint64_t* inc, uint64_t half_offset, int64_t row0,
                           int64_t rows, int32_t k, int8_t* out) {
  if (!state || !inc || !out || rows < 1 || k < 1 || row0 < 0) return fail(COFEM_EINVAL, "bad argument");
  CK(cudaSetDevice(device));
  int8_t* d = nullptr;
  CK(cudaMalloc(&d, (size_t)rows * k));
  const int64_t nchunk = (rows * k + 65) / 64 + 1;
  k_pcg64_rademacher<<<(int)std::min<int64_t>((nchunk + 255) / 256, 4096), 256>>>(state[0], state[1], inc[0], inc[1],
                                                                                 half_offset, row0, rows, k, d);
  cudaError_t e = cudaMemcpy(out, d, (size_t)rows * k, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(COFEM_ECUDA, cudaGetErrorString(e));
  return 0;
}

int cofem_bench_prepare(cofem_ctx* c, const double* y, double beta, const cofem_em_config* em,
                        const cofem_cg_config* cg, uint64_t dseed) {
  CKR(check_ctx(c));
  if (!y || !em || !cg) return fail(COFEM_EINVAL, "null argument");
  int rc = DISPATCH(c, em_prepare, c, y, beta, em, nullptr);
  if (rc) return rc;
  c->beta = beta;
  c->em = *em;
  c->cg = *cg;
  c->dseed = dseed;
  c->bench_iter = 0;
  c->bench_ready = true;
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int cofem_bench_iterations(cofem_ctx* c, int n_iter, int time_kernels, cofem_timing* out) {
  CKR(check_ctx(c));
  if (!c->bench_ready) return fail(COFEM_ESTATE, "cofem_bench_prepare first");
  c->time_kernels = time_kernels != 0;
  c->evnext = 0;
  c->timed.clear();
  c->ticks.clear();
  c->tick_prev = -1;
  c->ticks_on = time_kernels && c->kind == 2 && getenv("COFEM_TICKS");
  c->launches = c->fwd_launches = c->bwd_launches = c->pcg_steps = 0;
  c->ph_fwd_ms = c->ph_bwd_ms = 0;
  c->solve_launches = 0;
  CK(cudaEventRecord(c->t0, c->stream));
  for (int i = 0; i < n_iter; ++i) {
    cofem_cg_report rep;
    ++c->bench_iter;
    // never let the benchmark reach the final (non-updating) iteration
    const int t_total = c->bench_iter + 1;
    int rc = DISPATCH(c, em_iteration, c, c->bench_iter, t_total, c->beta, &c->em, &c->cg, nullptr, c->dseed, &rep);
    if (rc) return rc;
  }
  CK(cudaEventRecord(c->t1, c->stream));
  CK(cudaEventSynchronize(c->t1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, c->t0, c->t1));
  memset(out, 0, sizeof(*out));
  out->total_ms = ms;
  for (auto& tk : c->timed) {
    float d = 0;
    cudaEventElapsedTime(&d, c->evpool[tk.second], c->evpool[tk.second + 1]);
    if (tk.first == 0) out->fwd_ms += d;
    else if (tk.first == 1) out->bwd_ms += d;
    else out->solve_ms += d;
  }
  if (c->ticks_on) {  // live per-kernel times of the DCT step, kernels that ran (early exits excluded)
    static const char* names[] = {"row DCT-II", "column pass", "row DCT-III", "k_combine", "k_update(_psi)", "k_direction(_pap)"};
    double sum[6] = {0}, all = 0;
    long n[6] = {0};
    for (auto& tk : c->ticks) {
      float d = 0;
      cudaEventElapsedTime(&d, c->evpool[tk[1]], c->evpool[tk[2]]);
      if (d > 0.02f) sum[tk[0]] += d, n[tk[0]]++;
    }
    for (int i = 0; i < 6; ++i)
      if (n[i]) fprintf(stderr, "[ticks] %-18s n=%5ld avg %7.1f us\n", names[i], n[i], 1e3 * sum[i] / n[i]), all += sum[i] / n[i];
    fprintf(stderr, "[ticks] step (sum of averages) %7.1f us\n", 1e3 * all);
    c->ticks_on = false;
  }
  out->fwd_ms += c->ph_fwd_ms;  // contraction phases of persistent solves (globaltimer stamps)
  out->bwd_ms += c->ph_bwd_ms;
  out->solve_launches = c->solve_launches;
  out->fwd_launches = c->fwd_launches;
  out->bwd_launches = c->bwd_launches;
  out->pcg_steps = c->pcg_steps;
  out->kernel_launches = c->launches;
  c->time_kernels = false;
  return 0;
}

}  // extern "C"
