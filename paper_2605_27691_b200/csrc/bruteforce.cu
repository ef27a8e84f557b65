// bruteforce.cu -- exact k-NN spot check (K10): brute_force_knng
// evalio.cpp:125-147 for a set of query rows.  Bit-exact ids against the
// reference: exact-order distances, bottom-k by (dist, id), self excluded.
//
// CTA = 256 threads handles 32 queries; data rows stream through smem in
// tiles of 64 rows x 64 dims (cp.async 16 B), each thread keeps a 2x4
// register micro-tile of exact-order partial sums across the dim chunks; the
// 32x64 distance block lands in smem and each warp folds it into the running
// top-k of its 4 queries with warp-parallel knn_insert (core.cpp:99-112).
#include "refine_kernels.hpp"

namespace knng_b200 {
namespace {

constexpr int kBfThreads = 256;
constexpr int kBfQ = 32;
constexpr int kBfT = 64;
constexpr int kBfDC = 64;
constexpr int kBfDCP = kBfDC + 4;  // 68/4 = 17 odd

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <bool kCos>
__global__ __launch_bounds__(kBfThreads) void k_bruteforce(const float* __restrict__ X, u64 n,
                                                           int d, const u64* __restrict__ rows,
                                                           u64 q, u32 k, u32* __restrict__ out_ids,
                                                           float* __restrict__ out_d,
                                                           const float* __restrict__ nrm) {
  __shared__ __align__(16) float s_q[kBfQ * kBfDCP];
  __shared__ __align__(16) float s_x[kBfT * kBfDCP];
  __shared__ u64 s_dm[kBfQ][kBfT];
  __shared__ u64 s_qrow[kBfQ];
  const int tid = threadIdx.x;
  const unsigned lane = lane_id(), warp = tid >> 5;
  const u64 q0 = (u64)blockIdx.x * kBfQ;
  const int nq = (int)((q - q0) < (u64)kBfQ ? (q - q0) : (u64)kBfQ);
  if (tid < kBfQ) s_qrow[tid] = tid < nq ? rows[q0 + tid] : 0;
  u64 top[4] = {kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey};  // this warp's 4 queries
  const bool vec = (d & 3) == 0;
  // thread micro-tile: queries {qa, qa+16}, data rows {xb + 16c}
  const int qa = tid >> 4, xb = tid & 15;
  __syncthreads();
  for (u64 t0 = 0; t0 < n; t0 += kBfT) {
    const int nt = (int)((n - t0) < (u64)kBfT ? (n - t0) : (u64)kBfT);
    float acc[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0f;
    for (int c0 = 0; c0 < d; c0 += kBfDC) {
      const int dc = min(kBfDC, d - c0);
      __syncthreads();
      if (vec) {
        const int qd = dc >> 2;
        for (int t = tid; t < kBfQ * qd; t += kBfThreads) {
          const int row = t / qd, c4 = t - row * qd;
          cp_async16(s_q + row * kBfDCP + c4 * 4, X + s_qrow[row] * d + c0 + c4 * 4);
        }
        for (int t = tid; t < nt * qd; t += kBfThreads) {
          const int row = t / qd, c4 = t - row * qd;
          cp_async16(s_x + row * kBfDCP + c4 * 4, X + (t0 + row) * d + c0 + c4 * 4);
        }
        cp_async_wait_all();
      } else {
        for (int t = tid; t < kBfQ * dc; t += kBfThreads) {
          const int row = t / dc, c = t - row * dc;
          s_q[row * kBfDCP + c] = X[s_qrow[row] * d + c0 + c];
        }
        for (int t = tid; t < nt * dc; t += kBfThreads) {
          const int row = t / dc, c = t - row * dc;
          s_x[row * kBfDCP + c] = X[(t0 + row) * d + c0 + c];
        }
      }
      __syncthreads();
      const float* ra0 = s_q + qa * kBfDCP;
      const float* ra1 = s_q + (qa + 16) * kBfDCP;
      const float* rb[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) rb[c] = s_x + (xb + 16 * c) * kBfDCP;
      const int dc4 = dc & ~3;
      for (int dd = 0; dd < dc4; dd += 4) {
        const float4 a0 = *reinterpret_cast<const float4*>(ra0 + dd);
        const float4 a1 = *reinterpret_cast<const float4*>(ra1 + dd);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 b = *reinterpret_cast<const float4*>(rb[c] + dd);
          acc[0][c] = m_step4<kCos>(acc[0][c], a0, b);
          acc[1][c] = m_step4<kCos>(acc[1][c], a1, b);
        }
      }
      for (int dd = dc4; dd < dc; ++dd) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[0][c] = m_step<kCos>(acc[0][c], ra0[dd], rb[c][dd]);
          acc[1][c] = m_step<kCos>(acc[1][c], ra1[dd], rb[c][dd]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int qi = qa + 16 * r;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int xi = xb + 16 * c;
        const u64 row = t0 + xi;
        u64 key = kEmptyKey;
        if (xi < nt && qi < nq && row != s_qrow[qi])
          key = pack_key(m_finish<kCos>(acc[r][c], kCos ? nrm[s_qrow[qi]] : 0.0f,
                                        kCos ? nrm[row] : 0.0f),
                         (u32)row);
        s_dm[qi][xi] = key;
      }
    }
    __syncthreads();
    // fold into the running top-k, 4 queries per warp
    for (int qq = 0; qq < 4; ++qq) {
      const int qi = warp * 4 + qq;
      if (qi >= nq) continue;
      u64 rk = top[qq];
      u64 last = __shfl_sync(kFull, rk, k - 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const u64 c = s_dm[qi][h * 32 + lane];
        unsigned mask = __ballot_sync(kFull, c < last);
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const u64 cv = __shfl_sync(kFull, c, src);
          if (cv >= last) continue;
          const u32 pos = __popc(__ballot_sync(kFull, lane < k && rk < cv));
          const u64 up = __shfl_up_sync(kFull, rk, 1);
          if (lane > pos && lane < k) rk = up;
          if (lane == pos) rk = cv;
          last = __shfl_sync(kFull, rk, k - 1);
        }
      }
      top[qq] = rk;
    }
  }
  __syncthreads();
  for (int qq = 0; qq < 4; ++qq) {
    const int qi = warp * 4 + qq;
    if (qi >= nq) continue;
    const u64 rk = top[qq];
    if (lane < k) {
      out_ids[(q0 + qi) * k + lane] = key_id(rk);
      out_d[(q0 + qi) * k + lane] = key_dist(rk);
    }
  }
}

// Per-row norm chain of cosine_t (core.hpp:44-49): na = sum x*x in index
// order, no FMA.  One thread per row (a one-off O(N d) pass before a build or
// search; each row's 16-byte loads stay within its own lines).
__global__ void k_row_norms(const float* __restrict__ X, u64 n, int d, float* __restrict__ out) {
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
    const float* x = X + r * (u64)d;
    float acc = 0.0f;
    int i = 0;
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0)
      for (; i < d; i += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x + i));
        acc = dot_step4(acc, v, v);
      }
    for (; i < d; ++i) acc = dot_step(acc, x[i], x[i]);
    out[r] = acc;
  }
}

}  // namespace

void row_norms_device(const Runner& r, const float* X, uint64_t n, int d, float* out) {
  if (!n) return;
  DeviceGuard guard(r.device);
  const unsigned g = (unsigned)std::min<u64>(ceil_div<u64>(n, 256), (u64)r.num_sms * 32);
  k_row_norms<<<g, 256, 0, r.stream>>>(X, n, d, out);
  KNNG_LAUNCH_CHECK();
}

void brute_force_rows_device(Runner& r, const float* X, uint64_t n, int d, const uint64_t* rows,
                             uint64_t q, uint32_t k, uint32_t* out_ids, float* out_d,
                             const float* nrm) {
  require(k >= 1 && k < n, "brute_force_knng: k must be < N");
  require(k <= 32, "brute_force_knng: the B200 path supports k <= 32");
  if (!q) return;
  DeviceGuard guard(r.device);
  const unsigned g = (unsigned)ceil_div<u64>(q, kBfQ);
  if (nrm)
    k_bruteforce<true><<<g, kBfThreads, 0, r.stream>>>(X, n, d, rows, q, k, out_ids, out_d, nrm);
  else
    k_bruteforce<false><<<g, kBfThreads, 0, r.stream>>>(X, n, d, rows, q, k, out_ids, out_d, nrm);
  KNNG_LAUNCH_CHECK();
}

}  // namespace knng_b200
