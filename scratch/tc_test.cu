// Standalone probe of the tcgen05 int8 path: one CTA, TMA (SWIZZLE_64B) -> smem,
// tcgen05.mma kind::i8 into TMEM, tcgen05.ld back, checked against a CPU GEMM.
// mode 0: A K-major (A[m][k] row-major, 128 x K), B K-major (B[n][k], N x K)
// mode 1: A MN-major (At[k][m] row-major, K x 128)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n}\n" ::"r"(smem_u32(b)), "r"(parity));
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)layout << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1)
tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int32_t* out,
          int N, int K, int mode, int a_signed, int b_signed) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = sm;                 // 128 x K bytes (K-major) or K x 128 (MN-major, two 64-col blocks)
  unsigned char* sB = sm + 128 * K;       // N x K bytes
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (threadIdx.x == 0) {
    const uint32_t bytes = 128 * K + N * K;
    mbar_expect_tx(&bar_full, bytes);
    for (int kb = 0; kb < K / 64; ++kb) {
      if (mode == 0) {
        tma_load_3d(sA + kb * 128 * 64, &mapA, &bar_full, kb * 64, 0, 0);      // box {64, 128, 1}
      } else {
        // At[k][m]: box {64 m-bytes, 64 k-rows}; two m halves
        tma_load_3d(sA + kb * 2 * 4096, &mapA, &bar_full, 0, kb * 64, 0);
        tma_load_3d(sA + kb * 2 * 4096 + 4096, &mapA, &bar_full, 64, kb * 64, 0);
      }
      tma_load_3d(sB + kb * N * 64, &mapB, &bar_full, kb * 64, 0, 0);          // box {64, N, 1}
    }
  }
  if (threadIdx.x == 32) {
    mbar_wait(&bar_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // idesc: c=S32 (2) bits 4-5, a_format bit7-9, b_format 10-12, a_major 15, b_major 16, n>>3 @17, m>>4 @24
    uint32_t idesc = (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) | ((uint32_t)mode << 15) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int kb = 0; kb < K / 64; ++kb) {
      for (int kk = 0; kk < 2; ++kk) {
        uint64_t da, db;
        if (mode == 0) {
          da = make_desc(smem_u32(sA + kb * 128 * 64) + kk * 32, 16, 512, 4);
        } else {
          da = make_desc(smem_u32(sA + kb * 2 * 4096) + kk * 32 * 64, 4096, 512, 4);
        }
        db = make_desc(smem_u32(sB + kb * N * 64) + kk * 32, 16, 512, 4);
        const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
            ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar_mma)));
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32 lanes, N columns in chunks of 32
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 32 && c0 + j < N; ++j) out[row * N + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (EncodeFn)fn;
}

static void make_map(EncodeFn enc, CUtensorMap* m, void* ptr, uint64_t inner, uint64_t rows, uint32_t box0,
                     uint32_t box1) {
  cuuint64_t dims[3] = {inner, rows, 1};
  cuuint64_t strides[2] = {inner, inner * rows};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

int main() {
  EncodeFn enc = get_encode();
  const int N = 96, K = 128;
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int as = 0; as < 2; ++as)
      for (int bs = 0; bs < 2; ++bs) {
        std::vector<uint8_t> A(128 * K), B(N * K);  // logical A[m][k], B[n][k]
        srand(mode * 7 + as * 3 + bs);
        for (auto& v : A) v = rand() & 255;
        for (auto& v : B) v = rand() & 255;
        std::vector<uint8_t> Astore(128 * K);
        if (mode == 0) Astore = A;
        else for (int m = 0; m < 128; ++m) for (int k = 0; k < K; ++k) Astore[k * 128 + m] = A[m * K + k];
        uint8_t *dA, *dB; int32_t* dO;
        CK(cudaMalloc(&dA, Astore.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dO, 128 * N * 4));
        CK(cudaMemcpy(dA, Astore.data(), Astore.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
        CUtensorMap mA, mB;
        if (mode == 0) make_map(enc, &mA, dA, K, 128, 64, 128);
        else make_map(enc, &mA, dA, 128, K, 64, 64);
        make_map(enc, &mB, dB, K, N, 64, N);
        const int smem = 128 * K + N * K + 1024;
        CK(cudaFuncSetAttribute(tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        tc_kernel<<<1, 128, smem>>>(mA, mB, dO, N, K, mode, as, bs);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<int32_t> O(128 * N);
        CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < N; ++n) {
            long long s = 0;
            for (int k = 0; k < K; ++k) {
              int a = as ? (int)(int8_t)A[m * K + k] : (int)A[m * K + k];
              int b = bs ? (int)(int8_t)B[n * K + k] : (int)B[n * K + k];
              s += (long long)a * b;
            }
            if (s != O[m * N + n]) { if (bad < 3) printf("  m=%d n=%d got %d want %lld\n", m, n, O[m * N + n], s); ++bad; }
          }
        printf("mode %d a_signed %d b_signed %d: %s (%d bad)\n", mode, as, bs, bad ? "FAIL" : "ok", bad);
        fails += bad ? 1 : 0;
        cudaFree(dA); cudaFree(dB); cudaFree(dO);
      }
  return fails;
}
