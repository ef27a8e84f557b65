// join_tc.cu -- the NN-Descent local join (nndescent.cpp:135-197) on the
// 5th-generation tensor cores.
//
// Per point p the join evaluates sigma over new x new (i < j) and new x old
// pairs of p's join list and offers every pair passing `dist < worst` to both
// endpoints (nndescent.cpp:157-171).  Here the distances that DECIDE are
// bounds from a Gram matrix on the tensor cores; the distances that are
// STORED stay exact: k_apply recomputes the exact-order distance
// (core.hpp:23-30) of every candidate it may insert (nndescent.cu), so every
// graph entry is bit-identical to the reference's recomputation.
//
//   tile     128 rows = the join lists of several whole points (packed in
//            order; a point's list is <= 2B + k + B <= 128 rows)
//   producer warp 0: forms tiles from the chunk's active points, gathers the
//            tile's feature rows with TMA tile::gather4 (4 rows x 128 B per
//            instruction) into SWIZZLE_128B K-major panels of 32 dims,
//            completion on an mbarrier (expect_tx)
//   centering warps 2-3: subtract the joining point's vector from each of its
//            rows in smem (a' = a - p, exact fp32 subtraction) and accumulate
//            |a'|^2 -- the rows of a list are p's neighbours, so |a'| ~ the
//            distances being compared and the tf32 Gram error stays a small
//            fraction of them (data-independent precision)
//   MMA warp 1: tcgen05.mma.cta_group::1.kind::tf32, M = N = 128, G = A' A'^T
//            accumulated over the K panels into one of two TMEM accumulators
//   epilogue warps 4-7 (TMEM lane quarter = warp % 4): tcgen05.ld a row of G,
//            d2 = |a'|^2 + |b'|^2 - 2 G_ab for the pairs of the row's point,
//            lower bound lb2 = d2 - 2^-8 (|a'|^2 + |b'|^2) (>= 4x the measured
//            worst tf32 Gram error, profiles/r02_tc_probe.log), and offers
//            (u, v, sqrt(lb2)) whenever lb2 < worst^2: a superset of the
//            reference's offers, keyed by a lower bound of the exact distance
//            (k_apply recomputes every candidate whose bound beats the row).
// Pipelines: smem stages (full -> centred -> empty), two TMEM accumulators
// (full/empty), tile metadata slots (full via stage 0, empty) -- all mbarriers,
// no CTA-wide barrier after the prologue.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "join.hpp"
#include "nndescent.hpp"

namespace knng_b200 {
namespace {

constexpr int kTR = 128;                 // rows per tile (UMMA M = N)
constexpr int kPanelBytes = kTR * 128;   // one K panel: 128 rows x 32 fp32 (128 B), SW128
constexpr int kPPS = 4;                  // panels per smem stage
constexpr int kStageBytes = kPPS * kPanelBytes;
constexpr int kNS = 3;                   // smem stages
constexpr int kNM = 4;                   // tile metadata slots
constexpr int kMaxPts = kTR / 2;         // points per tile (every point has >= 2 rows)
constexpr int kThreads = 256;
constexpr int kXformWarps = 2;           // warps 2, 3
constexpr int kEpiWarp0 = 4;             // warps 4..7
constexpr int G = kJoinChunk;

struct TileMeta {
  int rows;    // staged rows (-1: end of work)
  int chunk;   // queue region
  int npts;
  int pad_;
  u32 rid[kTR];       // dataset row of tile row r
  float w2[kTR];      // worst[rid]^2 (+ rounding slack)
  float nrm[kTR];     // |a' - p|^2, written by the centering warps
  uint8_t seg_lo[kTR], new_end[kTR], seg_end[kTR], pidx[kTR];
  u32 pid[kMaxPts];   // joining point of each of the tile's points
};

struct ChunkState {  // producer-private
  u32 pt[G];
  u32 cnt[G];
};

struct SmemTC {
  unsigned char* stage;  // kNS x kStageBytes, 1024-aligned
  TileMeta* meta;        // kNM
  ChunkState* cs;
  uint64_t* bar;         // full[kNS], xdone[kNS], empty[kNS], tfull[2], tempty[2], mempty[kNM]
  u32* tslot;
  int* misc;
};

__host__ __device__ constexpr size_t tc_smem_bytes() {
  return 1024 + (size_t)kNS * kStageBytes + kNM * sizeof(TileMeta) + sizeof(ChunkState) +
         (3 * kNS + 4 + kNM) * 8 + 64;
}

__device__ __forceinline__ SmemTC carve_tc(unsigned char* raw) {
  SmemTC s;
  unsigned char* base = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  s.stage = base;
  unsigned char* p = base + (size_t)kNS * kStageBytes;
  s.meta = reinterpret_cast<TileMeta*>(p);
  p += kNM * sizeof(TileMeta);
  s.cs = reinterpret_cast<ChunkState*>(p);
  p += sizeof(ChunkState);
  p = (unsigned char*)(((uintptr_t)p + 7) & ~(uintptr_t)7);
  s.bar = reinterpret_cast<uint64_t*>(p);
  p += (3 * kNS + 4 + kNM) * 8;
  s.tslot = reinterpret_cast<u32*>(p);
  s.misc = reinterpret_cast<int*>(p + 16);
  return s;
}

__device__ __forceinline__ uint64_t* bar_full(const SmemTC& s, int i) { return s.bar + i; }
__device__ __forceinline__ uint64_t* bar_xdone(const SmemTC& s, int i) { return s.bar + kNS + i; }
__device__ __forceinline__ uint64_t* bar_empty(const SmemTC& s, int i) { return s.bar + 2 * kNS + i; }
__device__ __forceinline__ uint64_t* bar_tfull(const SmemTC& s, int i) { return s.bar + 3 * kNS + i; }
__device__ __forceinline__ uint64_t* bar_tempty(const SmemTC& s, int i) {
  return s.bar + 3 * kNS + 2 + i;
}
__device__ __forceinline__ uint64_t* bar_mempty(const SmemTC& s, int i) {
  return s.bar + 3 * kNS + 4 + i;
}

__device__ __forceinline__ unsigned su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int col, u32 r0, u32 r1,
                                        u32 r2, u32 r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
      : "memory");
}
// K-major SWIZZLE_128B operand descriptor: SBO = 1024 B (8-row atom), LBO = 1,
// version 1 (sm_100), layout type 2 (mma_sm100_desc.hpp SmemDescriptor).
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t a = su32(p);
  return ((a & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// kind::tf32, D f32, A/B tf32 K-major, N = M = 128 (InstrDescriptor bit layout)
constexpr unsigned kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(kTR >> 3) << 17) |
                            ((unsigned)(kTR >> 4) << 24);

__device__ __forceinline__ void mma_tf32(unsigned tmem, uint64_t da, uint64_t db, unsigned acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(b))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(unsigned addr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

struct TcArgs {
  const float* X;
  int d;
  int panels;          // ceil(d / 32)
  int stages;          // ceil(panels / kPPS)
  const u32* L_ids;
  const u32* L_cnt;
  int RMAX;
  const float* worst;
  const u32* act;
  u64 p_lo, p_hi;
  const u64* n_live;
  u32* chunk_counter;
  u64* q_key;
  u32* q_tgt;
  u32* q_fill;         // per chunk, zeroed before the launch, atomically grown
  u64 q_per_chunk;
  u64* counters;
};

// ---------------------------------------------------------------------------
// producer: next chunk -> tiles
// ---------------------------------------------------------------------------
__device__ int grab_chunk(const TcArgs& a, const SmemTC& s, int* np_out, u32* chunk_out) {
  const unsigned lane = lane_id();
  u32 chunk = 0;
  if (lane == 0) chunk = atomicAdd(a.chunk_counter, 1u);
  chunk = __shfl_sync(kFull, chunk, 0);
  u64 p_hi = a.p_hi;
  if (a.n_live) {
    const u64 live = *a.n_live;
    if (live < p_hi) p_hi = live;
  }
  const u64 p0 = a.p_lo + (u64)chunk * G;
  if (p0 >= p_hi) return 0;
  const int np = (p_hi - p0) < (u64)G ? (int)(p_hi - p0) : G;
  if ((int)lane < np) {
    const u32 pt = a.act ? a.act[p0 + lane] : (u32)(p0 + lane);
    s.cs->pt[lane] = pt;
    s.cs->cnt[lane] = a.L_cnt[pt];
  }
  __syncwarp();
  *np_out = np;
  *chunk_out = chunk;
  return 1;
}

__global__ __launch_bounds__(kThreads, 1) void k_join_tc(const __grid_constant__ CUtensorMap tm,
                                                         const TcArgs a) {
  extern __shared__ unsigned char smem_raw[];
  const SmemTC s = carve_tc(smem_raw);
  const int warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(bar_full(s, i), 1);
      mbar_init(bar_xdone(s, i), kXformWarps);
      mbar_init(bar_empty(s, i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_tfull(s, i), 1);
      mbar_init(bar_tempty(s, i), 4);
    }
    for (int i = 0; i < kNM; ++i) mbar_init(bar_mempty(s, i), 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        su32(s.tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = *s.tslot;

  if (warp == 0) {
    // ===================== producer =====================
    u64 staged = 0;
    int np = 0, j = 0;
    u32 chunk = 0;
    bool have = grab_chunk(a, s, &np, &chunk);
    for (u32 t = 0;; ++t) {
      const int ms = (int)(t % kNM);
      mbar_wait(bar_mempty(s, ms), ((t / kNM) & 1) ^ 1);
      TileMeta& M = s.meta[ms];
      // pack whole points of the current chunk (skipping points without pairs)
      int rows = 0, npts = 0;
      while (true) {
        if (have && j >= np) {
          if (rows > 0) break;  // tiles do not span chunks (per-chunk queue regions)
          have = grab_chunk(a, s, &np, &chunk);
          j = 0;
        }
        if (!have) break;
        const u32 c = s.cs->cnt[j];
        const int nn = (int)(c & 0xffff), na = (int)(c >> 16);
        if (nn == 0 || na < 2) {
          ++j;
          continue;
        }
        if (rows + na > kTR) break;
        const u32 pt = s.cs->pt[j];
        const u32* src = a.L_ids + (u64)pt * a.RMAX;
        for (int i = lane; i < na; i += 32) {
          const u32 id = src[i];
          const int r = rows + i;
          M.rid[r] = id;
          const float w = __ldg(a.worst + id);
          M.w2[r] = __fmul_ru(__fmul_ru(w, w), 1.0f + 3.0e-5f);
          M.seg_lo[r] = (uint8_t)rows;
          M.new_end[r] = (uint8_t)(rows + nn);
          M.seg_end[r] = (uint8_t)(rows + na);
          M.pidx[r] = (uint8_t)npts;
        }
        if (lane == 0) M.pid[npts] = pt;
        rows += na;
        ++npts;
        ++j;
      }
      const int rows_pad = (rows + 3) & ~3;
      for (int r = rows + lane; r < rows_pad; r += 32) M.rid[r] = M.rid[0];
      if (lane == 0) {
        M.rows = rows > 0 ? rows : -1;
        M.chunk = (int)chunk;
        M.npts = npts;
      }
      __syncwarp();
      staged += rows;
      // stages of this tile (the end marker takes one, without data)
      const int nst = rows > 0 ? a.stages : 1;
      for (int st = 0; st < nst; ++st) {
        const u32 g = t * (u32)a.stages + (u32)st;  // every tile owns a.stages stage uses
        const int slot = (int)(g % kNS);
        if (lane == 0) {
          mbar_wait(bar_empty(s, slot), ((g / kNS) & 1) ^ 1);
          if (rows > 0) {
            const int p0 = st * kPPS;
            const int pis = min(kPPS, a.panels - p0);
            mbar_expect_tx(bar_full(s, slot), (unsigned)(rows_pad * 128 * pis));
            unsigned char* sb = s.stage + (size_t)slot * kStageBytes;
            for (int r4 = 0; r4 < rows_pad; r4 += 4)
              for (int pp = 0; pp < pis; ++pp)
                gather4(sb + pp * kPanelBytes + r4 * 128, &tm, (p0 + pp) * 32, M.rid[r4],
                        M.rid[r4 + 1], M.rid[r4 + 2], M.rid[r4 + 3], bar_full(s, slot));
          } else {
            mbar_arrive(bar_full(s, slot));
          }
        }
        __syncwarp();
      }
      if (rows <= 0) break;
    }
    if (lane == 0 && a.counters)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + kCntStagedRows), staged);
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    for (u32 t = 0;; ++t) {
      const int acc = (int)(t & 1);
      const TileMeta& M = s.meta[t % kNM];
      bool end = false;
      for (int st = 0; st < a.stages; ++st) {
        const u32 g = t * (u32)a.stages + (u32)st;
        const int slot = (int)(g % kNS);
        mbar_wait(bar_xdone(s, slot), (g / kNS) & 1);
        if (st == 0 && M.rows < 0) {
          end = true;
          if (lane == 0) {
            mbar_arrive(bar_empty(s, slot));
            mbar_arrive(bar_tfull(s, acc));
          }
          break;
        }
        if (st == 0) mbar_wait(bar_tempty(s, acc), ((t >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const unsigned char* sb = s.stage + (size_t)slot * kStageBytes;
          const int pis = min(kPPS, a.panels - st * kPPS);
          for (int pp = 0; pp < pis; ++pp)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t dsc = sw128_desc(sb + pp * kPanelBytes + kk * 32);
              mma_tf32(tmem + (unsigned)(acc * kTR), dsc, dsc, (st | pp | kk) != 0);
            }
          mma_commit(bar_empty(s, slot));
          if (st == a.stages - 1) mma_commit(bar_tfull(s, acc));
        }
        __syncwarp();
      }
      if (end) break;
    }
  } else if (warp < kEpiWarp0) {
    // ===================== centering (a' = a - p) + |a'|^2 =====================
    const int tw = warp - 2;
    const int pp = (int)lane >> 3, cq = (int)lane & 7;  // panel, 16-B chunk of this lane
    for (u32 t = 0;; ++t) {
      TileMeta& M = s.meta[t % kNM];
      bool end = false;
      for (int st = 0; st < a.stages; ++st) {
        const u32 g = t * (u32)a.stages + (u32)st;
        const int slot = (int)(g % kNS);
        mbar_wait(bar_full(s, slot), (g / kNS) & 1);
        const int rows = M.rows;
        if (rows < 0) {
          end = true;
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_xdone(s, slot));
          break;
        }
        unsigned char* sb = s.stage + (size_t)slot * kStageBytes;
        const int dim = (st * kPPS + pp) * 32 + cq * 4;
        const bool live = pp < kPPS && dim < a.d;
        int cur_pt = -1;
        float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = tw; r < rows; r += kXformWarps) {
          const int pi = M.pidx[r];
          float part = 0.0f;
          if (live) {
            if (pi != cur_pt) {
              cur_pt = pi;
              pv = __ldg(reinterpret_cast<const float4*>(a.X + (u64)M.pid[pi] * a.d + dim));
            }
            float4* q = reinterpret_cast<float4*>(sb + pp * kPanelBytes + r * 128 +
                                                  ((cq ^ (r & 7)) << 4));
            float4 v = *q;
            v.x = __fsub_rn(v.x, pv.x);
            v.y = __fsub_rn(v.y, pv.y);
            v.z = __fsub_rn(v.z, pv.z);
            v.w = __fsub_rn(v.w, pv.w);
            *q = v;
            part = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, v.w * v.w)));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
          if (lane == 0) M.nrm[r] = st == 0 ? part : M.nrm[r] + part;
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_xdone(s, slot));
      }
      if (end) break;
    }
  } else {
    // ===================== epilogue: bounds -> offers =====================
    const int ew = warp - kEpiWarp0;  // TMEM lane quarter
    u64 my_pairs = 0, my_offers = 0;
    for (u32 t = 0;; ++t) {
      const int acc = (int)(t & 1);
      const int ms = (int)(t % kNM);
      const TileMeta& M = s.meta[ms];
      mbar_wait(bar_tfull(s, acc), (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int rows = M.rows;
      if (rows < 0) break;
      const int r = ew * 32 + (int)lane;
      const bool rv = r < rows && r < (int)M.new_end[r];
      const int hi_r = rv ? (int)M.seg_end[r] : 0;
      const float n_r = rv ? M.nrm[r] : 0.0f;
      const float w2_r = rv ? M.w2[r] : 0.0f;
      const u32 id_r = rv ? M.rid[r] : 0u;
      const int c_lo = __reduce_min_sync(kFull, rv ? (unsigned)(r + 1) : 0xffffu);
      const int c_hi = __reduce_max_sync(kFull, (unsigned)hi_r);
      const u32 chunk = (u32)M.chunk;
      u64* qk = a.q_key + (u64)chunk * a.q_per_chunk;
      u32* qt = a.q_tgt + (u64)chunk * a.q_per_chunk;
      for (int c0 = c_lo & ~15; c0 < c_hi; c0 += 16) {
        float gv[16];
        tmem_ld16(tmem + ((unsigned)(ew * 32) << 16) + (unsigned)(acc * kTR + c0), gv);
        u32 pass = 0;  // bit 2j: offer to r, bit 2j+1: offer to column c0+j
        float lb[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int c = c0 + jj;
          lb[jj] = 0.0f;
          if (rv && c > r && c < hi_r) {
            const float nc = M.nrm[c];
            const float sn = n_r + nc;
            const float d2 = fmaf(-2.0f, gv[jj], sn);
            const float lb2 = fmaxf(fmaf(-0.00390625f, sn, d2), 0.0f);
            lb[jj] = __fmul_rd(__fsqrt_rd(lb2), 0.99998f);
            if (lb2 < w2_r) pass |= 1u << (2 * jj);
            if (lb2 < M.w2[c]) pass |= 2u << (2 * jj);
            ++my_pairs;
          }
        }
        const int cnt = __popc(pass);
        const int tot = __reduce_add_sync(kFull, (unsigned)cnt);
        if (!tot) continue;
        u32 base = 0;
        if (lane == 0) base = atomicAdd(a.q_fill + chunk, (u32)tot);
        u32 slot = __shfl_sync(kFull, base, 0);
        my_offers += cnt;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const u32 two = (pass >> (2 * jj)) & 3u;
          if (!__any_sync(kFull, two != 0)) continue;
          const u32 idc = two ? M.rid[c0 + jj] : 0u;
#pragma unroll
          for (int dir = 0; dir < 2; ++dir) {
            const bool on = (two >> dir) & 1u;
            const unsigned mb = __ballot_sync(kFull, on);
            if (on) {
              const u32 at = slot + __popc(mb & lanemask_lt());
              qk[at] = pack_key(lb[jj], dir ? id_r : idc);
              qt[at] = dir ? idc : id_r;
            }
            slot += __popc(mb);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar_tempty(s, acc));
        mbar_arrive(bar_mempty(s, ms));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      my_pairs += __shfl_xor_sync(kFull, my_pairs, o);
      my_offers += __shfl_xor_sync(kFull, my_offers, o);
    }
    if (lane == 0 && a.counters) {
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + kCntPairs), my_pairs);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + kCntOffers), my_offers);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return (EncodeTiledFn)f;
  }();
  return fn;
}

}  // namespace

bool join_tc_supported(const float* X, int d, uint32_t k, uint32_t B, bool cosine) {
  // opt-in (KNNG_JOIN=tc): measured slower than the exact-order kernel on C2
  // (DESIGN.md section 4b), so the exact kernel is the default
  const char* v = std::getenv("KNNG_JOIN");
  if (!v || std::string(v) != "tc") return false;
  const uint32_t max_rows = 2 * B + k + B;
  return !cosine && X && d > 0 && (d % 4) == 0 && ((uintptr_t)X % 16) == 0 && max_rows <= kTR &&
         encode_fn() != nullptr;
}

void launch_join_tc(const Runner& r, const JoinPlan& plan, const JoinLaunch& l) {
  static thread_local int configured_dev = -1;
  const size_t smem = tc_smem_bytes();
  if (configured_dev != r.device) {
    KNNG_CUDA(cudaFuncSetAttribute(k_join_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    configured_dev = r.device;
  }
  CUtensorMap tm;
  const uint64_t n_rows = l.n_rows;
  cuuint64_t gdim[2] = {(cuuint64_t)l.d, (cuuint64_t)n_rows};
  cuuint64_t gstr[1] = {(cuuint64_t)l.d * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  const CUresult cr =
      encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(l.X), gdim, gstr,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(cr == CUDA_SUCCESS, "nn_descent: cuTensorMapEncodeTiled failed for the join");
  TcArgs a{};
  a.X = l.X;
  a.d = l.d;
  a.panels = (l.d + 31) / 32;
  a.stages = (a.panels + kPPS - 1) / kPPS;
  a.L_ids = l.L_ids;
  a.L_cnt = l.L_cnt;
  a.RMAX = plan.RMAX;
  a.worst = l.worst;
  a.act = l.act;
  a.p_lo = l.p_lo;
  a.p_hi = l.p_hi;
  a.n_live = l.n_live;
  a.chunk_counter = l.chunk_counter;
  a.q_key = l.q_key;
  a.q_tgt = l.q_tgt;
  a.q_fill = l.q_fill;
  a.q_per_chunk = plan.q_per_chunk;
  a.counters = l.counters;
  k_join_tc<<<(unsigned)r.num_sms, kThreads, smem, r.stream>>>(tm, a);
  KNNG_LAUNCH_CHECK();
}

}  // namespace knng_b200
