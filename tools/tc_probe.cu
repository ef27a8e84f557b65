// tc_probe.cu -- standalone check of the tcgen05 building blocks the TC join
// uses: TMA tile::gather4 of arbitrary rows into a SWIZZLE_128B K-major tile,
// tcgen05.mma kind::tf32 (M=128, N=128) Gram A.A^T into TMEM, tcgen05.ld back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/tc_probe tools/tc_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int col, int r0, int r1,
                                        int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

constexpr int D = 128, ROWS = 128, PANEL = ROWS * 128;

__global__ void probe(const __grid_constant__ CUtensorMap tm, const int* rows, float* G) {
  extern __shared__ unsigned char sm_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(base + 4 * PANEL);
  unsigned* tslot = (unsigned*)(base + 4 * PANEL + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = *tslot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, ROWS * D * 4);
    for (int p = 0; p < D / 32; ++p)
      for (int r = 0; r < ROWS; r += 4)
        gather4(base + p * PANEL + r * 128, &tm, p * 32, rows[r], rows[r + 1], rows[r + 2],
                rows[r + 3], bar);
  }
  mbar_wait(bar, 0);
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(ROWS >> 3) << 17) |
                           ((unsigned)(128 >> 4) << 24);
    for (int s = 0; s < D / 8; ++s) {
      const uint64_t ad = sw128_desc(base + (s / 4) * PANEL + (s % 4) * 32);
      const unsigned acc = s > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(ad), "l"(ad), "r"(idesc), "r"(acc));
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar + 1))
        : "memory");
  }
  mbar_wait(bar + 1, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c = 0; c < 128; c += 32) {
    unsigned v[32];
    const unsigned addr = tmem + ((unsigned)(warp * 32) << 16) + c;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) G[row * 128 + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  const int N = 5000;
  std::vector<float> X((size_t)N * D);
  srand(1);
  for (auto& v : X) v = (float)rand() / RAND_MAX * 10.0f - 5.0f;
  std::vector<int> rows(ROWS);
  for (int i = 0; i < ROWS; ++i) rows[i] = (i * 37 + 11) % N;
  float *dX, *dG;
  int* dR;
  CK(cudaMalloc(&dX, X.size() * 4));
  CK(cudaMalloc(&dG, ROWS * 128 * 4));
  CK(cudaMalloc(&dR, ROWS * 4));
  CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dR, rows.data(), ROWS * 4, cudaMemcpyHostToDevice));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)N};
  cuuint64_t gstr[1] = {(cuuint64_t)D * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  const int smem = 4 * PANEL + 1024 + 256;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(tm, dR, dG);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> G(ROWS * 128);
  CK(cudaMemcpy(G.data(), dG, G.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  int bad = 0;
  for (int i = 0; i < ROWS; ++i)
    for (int j = 0; j < 128; ++j) {
      double ref = 0, scale = 0;
      for (int t = 0; t < D; ++t) {
        ref += (double)X[(size_t)rows[i] * D + t] * X[(size_t)rows[j] * D + t];
        scale += fabs((double)X[(size_t)rows[i] * D + t] * X[(size_t)rows[j] * D + t]);
      }
      const double e = fabs(G[i * 128 + j] - ref) / scale;
      if (e > worst) worst = e;
      if (e > 4e-3) ++bad;
    }
  printf("tc_probe: max |G - ref| / sum|a_i b_i| = %.3e, bad = %d of %d; G[0][0]=%f G[5][77]=%f\n",
         worst, bad, ROWS * 128, G[0], G[5 * 128 + 77]);
  return bad ? 2 : 0;
}
