// fp32 mu-mode product GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32) with the
// three-pass split that recovers fp32 accuracy — the precision variant behind the paper's "CUDA
// single" columns (Table 5, Table 7).
//
// Every fp32 operand x is used as two tf32-valued parts, hi = rna_tf32(x) and
// lo = rna_tf32(x - hi) (|x - hi - lo| <= 2^-22 |x|).  A product is then
//     A B ~ A_lo B_hi + A_hi B_lo + A_hi B_hi          (3 tf32 MMAs, fp32 accumulate in TMEM)
// which drops only the A_lo B_lo term (~2^-22 relative).
//
// kind::tf32 reads both operands K-major only (measured: tools/tcgen05_probe.cu, an MN-major B
// yields zeros), while the mode products need no permutes: for mu >= 2 the tensor
// slab X_b is MN-major (n contiguous).  So the two operands take different routes:
//   * the "static" operand — the phi-matrix / L planes (A for mu >= 2, B = L^T for mu = 1) — is
//     split and laid out K-major once on the host side of a launch (or once per phi bank) and
//     TMA-loaded (128-B swizzle) straight into the MMA's shared-memory layout;
//   * the "tensor" operand is TMA-loaded raw (fp32) and converter warps split it into (hi, lo) in
//     the K-major 128-B-swizzled layout the MMA reads — transposing it for mu >= 2 on the way —
//     so tensors stay plain fp32 in HBM (4 B per element read, 4 B written).
//
// Structure (one CTA per SM, persistent over output tiles of 128 x 128, 320 threads):
//   warp 0      TMA producer: per k-tile the static planes (2 x 128 x 32) and the raw tensor tile;
//   warp 1      MMA issuer (one elected thread): 4 k-steps x 3 MMAs (M = N = 128, K = 8) per
//               k-tile into a FRESH TMEM accumulator (one of 4 x 128 columns) per k-tile;
//   warps 2..5  converters: raw tensor tile -> (hi, lo) K-major swizzled (double-buffered);
//   warps 6..9  accumulators + epilogue: every k-tile's partial is read back (tcgen05.ld, 32
//               lanes x 128 columns per warp) and added in fp32 round-to-nearest in registers
//               (one output row per thread); after the tile's last k-tile, C = alpha acc + beta D.
// The per-k-tile read-back is the accuracy fix measured in profiles/f32_accuracy_r02.json: the
// tensor core's fp32 accumulation is biased (its error grew linearly with K, 19x numpy's fp32
// sgemm at K = 1024), so the tensor core only ever sums K = 32 products (x3 passes) and the long
// sums are rounded to nearest.
#include "kx_internal.h"

#include <cuda.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace kx {
namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3, TCONV = 2;
constexpr int T_PLANE = 128 * TBK * 4;                 // 16 KB: one 128 x 32 fp32 tile
constexpr int T_STAGE_BYTES = 3 * T_PLANE;             // static hi, static lo, raw tensor
constexpr int T_CONV_BYTES = 2 * T_PLANE;              // converted tensor hi, lo
constexpr int T_EPI_BYTES = 4 * 32 * 32 * 4;            // per epilogue warp: one 32 x 32 fp32 store chunk
// stages | converted buffers | barriers (1 KB block) | epilogue store chunks (1 KB aligned) + alignment
constexpr int T_SMEM = TSTAGES * T_STAGE_BYTES + TCONV * T_CONV_BYTES + 1024 + T_EPI_BYTES + 1024;
constexpr int T_THREADS = 320;
constexpr int T_PSTRIDE = TBN + 4;                     // cluster split-K partial row (floats)
static_assert(TBM * T_PSTRIDE * 4 <= TSTAGES * T_STAGE_BYTES, "partial fits in the stage memory");
constexpr int T_KBUF = 4;                              // per-k-tile partial accumulators in TMEM
#ifndef KX_TF32_KPP
#define KX_TF32_KPP 2
#endif
constexpr int T_KPP = KX_TF32_KPP;                     // k-tiles summed in TMEM per partial
constexpr int T_TMEM_COLS = T_KBUF * TBN;              // 4 x 128 fp32 columns = all of TMEM

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra W_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}

// 5-D tiled TMA load into shared memory, completion counted on `bar` (bytes)
__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(bar))
      : "memory");
}

// tiled TMA store of a shared-memory box (5-D map, bulk-group completion)
__device__ __forceinline__ void tma_store5(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(0)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

// the same box added element-wise into global memory (TMA reduction, fp32 add, round to nearest)
__device__ __forceinline__ void tma_reduce_add5(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                                int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.5d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(0)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

// shared-memory matrix descriptor (tcgen05), K-major, 128-B swizzle: start, leading / stride
// byte offsets (16-B units), version 1 (sm_100), layout SWIZZLE_128B
__device__ __forceinline__ uint64_t sdesc(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;     // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: 8-row groups 1 KB apart
  d |= (uint64_t)1 << 46;             // version
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4)           // c_format F32
                            | (2u << 7)         // a_format TF32
                            | (2u << 10)        // b_format TF32
                            | ((uint32_t)(TBN >> 3) << 17) | ((uint32_t)(TBM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(unsigned tmem_d, uint64_t da, uint64_t db, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n"
      " setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split4(const float4 x, float4& h, float4& l) {
  h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
  l = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z), tf32_rna(x.w - h.w));
}

struct Tf32GemmArgs {
  CUtensorMap mapS_hi, mapS_lo, mapT;   // 64-B aligned members first
  CUtensorMap mapC[MAXS];               // output (n, m, t, b), 32 x 32 boxes, 128-B swizzle (tma_store)
  int kind, M, N, kseg, nseg, slo, ns, nt, nb, vec4;
  int csplit;   // > 1: cluster split-K — the S CTAs of a cluster share one tile's k-tiles
  int tile0, tile1;   // the launch covers tiles [tile0, tile1) of the z-major tile order
  float alpha, beta;
  int diag_nostore;   // diagnostics (KX_TF32_NOSTORE=1): skip the output stores
  int tma_store;      // 1: whole-chunk TMA stores of the output (mapC), else per-thread rows;
                      // 2: in place C += alpha acc (C == D, beta == 1) as TMA reduce-add boxes
  long long ldc, ldd, sC_t, sC_b, sD_t, sD_b;
  float* C[MAXS];
  const float* D[MAXS];
};

struct TileCoord {
  int m0, n0, s, t, b;
};

__device__ __forceinline__ TileCoord tile_coord(const Tf32GemmArgs& p, int tiles_m, int tiles_n, int tl) {
  const int tmn = tiles_m * tiles_n;
  const int z = tl / tmn, r = tl - z * tmn;
  TileCoord c;
  if (p.kind == TF32_COL) {   // m fastest: consecutive CTAs share the big tensor panel
    c.m0 = (r % tiles_m) * TBM;
    c.n0 = (r / tiles_m) * TBN;
  } else {                    // n fastest: consecutive CTAs share the tensor rows
    c.n0 = (r % tiles_n) * TBN;
    c.m0 = (r / tiles_n) * TBM;
  }
  c.b = z % p.nb;
  const int zt = z / p.nb;
  c.t = zt % p.nt;
  c.s = zt / p.nt;
  return c;
}

// Work items of a CTA in tiles [tile0, tile1): persistent over tiles (whole k range), or —
// cluster split-K — the one tile of its cluster and its 1/S share of the k-tiles.
template <bool SPLIT>
struct Work {
  int n, tl0, step, kb, ke;
  __device__ __forceinline__ Work(const Tf32GemmArgs& p, int ntiles, int ktiles) {
    if (SPLIT) {
      const int r = blockIdx.x % p.csplit;
      n = 1;
      tl0 = p.tile0 + blockIdx.x / p.csplit;
      step = 1;
      kb = r * ktiles / p.csplit;
      ke = (r + 1) * ktiles / p.csplit;
    } else {
      tl0 = p.tile0 + blockIdx.x;
      step = gridDim.x;
      const int end = min(ntiles, p.tile1);
      n = tl0 < end ? (end - 1 - tl0) / step + 1 : 0;
      kb = 0;
      ke = ktiles;
    }
  }
};

// K-major 128-B-swizzled byte offset of element k (< 32) of row r (< 128) of a 128 x 32 tile
__device__ __forceinline__ unsigned kmajor_off(unsigned r, unsigned kchunk) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((kchunk ^ (r & 7)) << 4);
}

template <bool SPLIT>
__global__ void __launch_bounds__(T_THREADS, 1) tf32x3_gemm_kernel(const __grid_constant__ Tf32GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* conv = smem + TSTAGES * T_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(conv + TCONV * T_CONV_BYTES);
  uint64_t* empty = full + TSTAGES;
  uint64_t* cfull = empty + TSTAGES;    // converted tensor buffer ready (converters -> MMA)
  uint64_t* cempty = cfull + TCONV;     // converted buffer read by the MMAs (MMA -> converters)
  uint64_t* kfull = cempty + TCONV;     // k-tile partial ready (MMA -> accumulator warps)
  uint64_t* kempty = kfull + T_KBUF;    // partial read back (accumulator warps -> MMA)
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(kempty + T_KBUF);
  float* epi = reinterpret_cast<float*>(conv + TCONV * T_CONV_BYTES + 1024);   // 1 KB aligned store chunks

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (p.M + TBM - 1) / TBM, tiles_n = (p.N + TBN - 1) / TBN;
  const int ntiles = tiles_m * tiles_n * p.ns * p.nt * p.nb;
  const int kps = (p.kseg + TBK - 1) / TBK;
  const int ktiles = kps * p.nseg;
  const bool col = p.kind == TF32_COL;

  if (threadIdx.x == 0) {
    for (int i = 0; i < TSTAGES; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1 + 4);   // the MMAs' commit + the 4 converter warps
    }
    for (int i = 0; i < TCONV; ++i) {
      mbar_init(cfull + i, 4);
      mbar_init(cempty + i, 1);
    }
    for (int i = 0; i < T_KBUF; ++i) {
      mbar_init(kfull + i, 1);
      mbar_init(kempty + i, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {   // TMEM allocation (this warp also frees it)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "n"(T_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const unsigned tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      const Work<SPLIT> wk(p, ntiles, ktiles);
      for (int w = 0; w < wk.n; ++w) {
        const TileCoord c = tile_coord(p, tiles_m, tiles_n, wk.tl0 + w * wk.step);
        for (int kt = wk.kb; kt < wk.ke; ++kt, ++it) {
          const int st = it % TSTAGES, fill = it / TSTAGES;
          if (fill > 0) mbar_wait(empty + st, (fill - 1) & 1);
          uint8_t* sS = smem + st * T_STAGE_BYTES;
          mbar_expect_tx(full + st, T_STAGE_BYTES);
          const int seg = kt / kps, k0 = (kt - seg * kps) * TBK;
          if (col) {
            // static A (k, m, t, s); tensor B raw (n, k, b, t, s), one 128 x 32 box
            tma_load5(sS, &p.mapS_hi, k0, c.m0, c.t, c.s, 0, full + st);
            tma_load5(sS + T_PLANE, &p.mapS_lo, k0, c.m0, c.t, c.s, 0, full + st);
            tma_load5(sS + 2 * T_PLANE, &p.mapT, c.n0, k0, c.b, c.t, c.s, full + st);
          } else {
            // static B (k, n, seg, s); tensor A raw (k, m, seg % slo, seg / slo, s)
            const int shi = seg / p.slo;
            tma_load5(sS, &p.mapS_hi, k0, c.n0, seg, c.s, 0, full + st);
            tma_load5(sS + T_PLANE, &p.mapS_lo, k0, c.n0, seg, c.s, 0, full + st);
            tma_load5(sS + 2 * T_PLANE, &p.mapT, k0, c.m0, seg - shi * p.slo, shi, c.s, full + st);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int it = 0;
    const Work<SPLIT> wk(p, ntiles, ktiles);
    int pt = 0;   // partials started
    for (int w = 0; w < wk.n; ++w) {
      for (int kt = wk.kb; kt < wk.ke; ++kt, ++it) {
        const int st = it % TSTAGES, cb = it % TCONV;
        const bool first = (kt - wk.kb) % T_KPP == 0;
        const bool last = (kt - wk.kb) % T_KPP == T_KPP - 1 || kt + 1 == wk.ke;
        const int kb = (first ? pt : pt - 1) % T_KBUF;
        if (first) {
          if (pt >= T_KBUF) mbar_wait(kempty + kb, ((pt / T_KBUF) - 1) & 1);   // partial read back
          ++pt;
        }
        mbar_wait(full + st, (it / TSTAGES) & 1);
        mbar_wait(cfull + cb, (it / TCONV) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const unsigned tmem_d = tmem_base + kb * TBN;
          const unsigned s_hi = su32(smem + st * T_STAGE_BYTES), s_lo = s_hi + T_PLANE;
          const unsigned t_hi = su32(conv + cb * T_CONV_BYTES), t_lo = t_hi + T_PLANE;
          // COL: A = static, B = converted tensor;  ROW: A = converted tensor, B = static
          const unsigned a_hi = col ? s_hi : t_hi, a_lo = col ? s_lo : t_lo;
          const unsigned b_hi = col ? t_hi : s_hi, b_lo = col ? t_lo : s_lo;
#pragma unroll
          for (int ks = 0; ks < TBK / 8; ++ks) {   // k-step = 32 B inside the 128-B swizzled rows
            mma_tf32(tmem_d, sdesc(a_lo + ks * 32), sdesc(b_hi + ks * 32), (ks > 0 || !first) ? 1u : 0u);
            mma_tf32(tmem_d, sdesc(a_hi + ks * 32), sdesc(b_lo + ks * 32), 1u);
            mma_tf32(tmem_d, sdesc(a_hi + ks * 32), sdesc(b_hi + ks * 32), 1u);
          }
          mma_commit(empty + st);    // static planes free once these MMAs finish
          mma_commit(cempty + cb);   // converted buffer free
          if (last) mma_commit(kfull + kb);    // this partial (kpp k-tiles) complete
        }
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ converters (warps 2..5)
    const int ct = threadIdx.x - 64;   // 0..127
    int it = 0;
    const Work<SPLIT> wk(p, ntiles, ktiles);
    for (int w = 0; w < wk.n; ++w) {
      for (int kt = wk.kb; kt < wk.ke; ++kt, ++it) {
        const int st = it % TSTAGES, cb = it % TCONV;
        mbar_wait(full + st, (it / TSTAGES) & 1);
        if (it >= TCONV) mbar_wait(cempty + cb, ((it / TCONV) - 1) & 1);
        const uint8_t* raw = smem + st * T_STAGE_BYTES + 2 * T_PLANE;
        uint8_t* ohi = conv + cb * T_CONV_BYTES;
        uint8_t* olo = ohi + T_PLANE;
        if (col) {
          // raw MN-major [k][n] (512-B rows, unswizzled) -> K-major row n = ct, 8 chunks of 4 k
          const float* r = reinterpret_cast<const float*>(raw);
#pragma unroll
          for (int kc = 0; kc < TBK / 4; ++kc) {
            const float4 x = make_float4(r[(4 * kc + 0) * TBN + ct], r[(4 * kc + 1) * TBN + ct],
                                         r[(4 * kc + 2) * TBN + ct], r[(4 * kc + 3) * TBN + ct]);
            float4 h, l;
            split4(x, h, l);
            const unsigned o = kmajor_off(ct, kc);
            *reinterpret_cast<float4*>(ohi + o) = h;
            *reinterpret_cast<float4*>(olo + o) = l;
          }
        } else {
          // raw already K-major 128-B swizzled (TMA): elementwise split in place of layout
#pragma unroll
          for (int i = 0; i < T_PLANE / 16 / 128; ++i) {
            const unsigned o = (ct + 128 * i) * 16;
            float4 h, l;
            split4(*reinterpret_cast<const float4*>(raw + o), h, l);
            *reinterpret_cast<float4*>(ohi + o) = h;
            *reinterpret_cast<float4*>(olo + o) = l;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> MMA reads
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(cfull + cb);
          mbar_arrive(empty + st);   // raw tile consumed
        }
      }
    }
  } else {
    // ------------------------------------------------------------ accumulate + epilogue (warps 6..9)
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    int it = 0;
    const Work<SPLIT> wk(p, ntiles, ktiles);
    for (int w = 0; w < wk.n; ++w) {
      const TileCoord c = tile_coord(p, tiles_m, tiles_n, wk.tl0 + w * wk.step);
      float acc[TBN];
#pragma unroll
      for (int j = 0; j < TBN; ++j) acc[j] = 0.0f;
      for (int kt = wk.kb; kt < wk.ke; kt += T_KPP, ++it) {   // it: partials read back
        const int kb = it % T_KBUF;
        mbar_wait(kfull + kb, (it / T_KBUF) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
        for (int cb = 0; cb < TBN; cb += 32) {
          unsigned v[32];
          const unsigned taddr = tmem_base + ((unsigned)(q * 32) << 16) + kb * TBN + cb;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[cb + j] = __fadd_rn(acc[cb + j], __uint_as_float(v[j]));
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(kempty + kb);   // partial buffer free for the MMAs
      }
      if constexpr (SPLIT) {
        // cluster split-K: park this CTA's partial (row per thread) in the now idle stage
        // memory, then every CTA sums its 1/S of the rows over the cluster's partials in rank
        // (= k) order through distributed shared memory and stores them (deterministic)
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        float* part = reinterpret_cast<float*>(smem);
        const int row = q * 32 + lane;
#pragma unroll
        for (int j = 0; j < TBN; j += 4)
          *reinterpret_cast<float4*>(part + row * T_PSTRIDE + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        cl.sync();
        const int S = p.csplit, r = (int)cl.block_rank(), col = threadIdx.x - 192;   // 0..127
        const int rows = TBM / S;
        for (int i = 0; i < rows; ++i) {
          const int rr = r * rows + i;
          float v = 0.0f;
          for (int j = 0; j < S; ++j) v = __fadd_rn(v, cl.map_shared_rank(part, j)[rr * T_PSTRIDE + col]);
          const int mm = c.m0 + rr, nn = c.n0 + col;
          if (mm < p.M && nn < p.N) {
            float o = p.alpha * v;
            const float* D = p.D[c.s];
            if (D) o += p.beta * D[c.t * p.sD_t + c.b * p.sD_b + (long long)mm * p.ldd + nn];
            p.C[c.s][c.t * p.sC_t + c.b * p.sC_b + (long long)mm * p.ldc + nn] = o;
          }
        }
        cl.sync();   // no CTA leaves while its partial may still be read
        continue;
      }
      if (p.diag_nostore) continue;
      const int m = c.m0 + q * 32 + lane;
      const long long oc = c.t * p.sC_t + c.b * p.sC_b + (long long)m * p.ldc + c.n0;
      const long long od = c.t * p.sD_t + c.b * p.sD_b + (long long)m * p.ldd + c.n0;
      float* C = p.C[c.s];
      const float* D = p.D[c.s];
      if (p.tma_store) {
        // this warp's 32 rows go out as four 32 x 32 boxes: each thread writes its row's 32
        // values into the 128-B-swizzled chunk (16-B pieces XOR row: conflict-free), one lane
        // issues the TMA store; the chunk is rewritten only after that store has read it.
        // Out-of-range rows / columns are clipped by the TMA unit.
        float* stg = epi + q * (32 * 32);
        const bool dl = D && m < p.M && p.tma_store == 1;
#pragma unroll
        for (int cb = 0; cb < TBN; cb += 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[cb + j] *= p.alpha;   // in place: no extra registers
          if (dl) {   // tma_store implies vec4: a float4 of D is wholly inside or outside N
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (c.n0 + cb + 4 * j < p.N) {
                const float4 dd = *reinterpret_cast<const float4*>(D + od + cb + 4 * j);
                acc[cb + 4 * j] += p.beta * dd.x;
                acc[cb + 4 * j + 1] += p.beta * dd.y;
                acc[cb + 4 * j + 2] += p.beta * dd.z;
                acc[cb + 4 * j + 3] += p.beta * dd.w;
              }
            }
          }
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(stg + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                make_float4(acc[cb + 4 * j], acc[cb + 4 * j + 1], acc[cb + 4 * j + 2], acc[cb + 4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (p.tma_store == 2) tma_reduce_add5(&p.mapC[c.s], stg, c.n0 + cb, c.m0 + q * 32, c.t, c.b);
            else tma_store5(&p.mapC[c.s], stg, c.n0 + cb, c.m0 + q * 32, c.t, c.b);
          }
        }
        continue;
      }
      if (m >= p.M) continue;
      if (c.n0 + TBN <= p.N && p.vec4) {
#pragma unroll
        for (int j = 0; j < TBN; j += 4) {
          float4 r = make_float4(p.alpha * acc[j], p.alpha * acc[j + 1], p.alpha * acc[j + 2], p.alpha * acc[j + 3]);
          if (D) {
            const float4 dd = *reinterpret_cast<const float4*>(D + od + j);
            r.x += p.beta * dd.x;
            r.y += p.beta * dd.y;
            r.z += p.beta * dd.z;
            r.w += p.beta * dd.w;
          }
          *reinterpret_cast<float4*>(C + oc + j) = r;
        }
      } else {
#pragma unroll
        for (int j = 0; j < TBN; ++j) {
          if (c.n0 + j < p.N) {
            float r = p.alpha * acc[j];
            if (D) r += p.beta * D[od + j];
            C[oc + j] = r;
          }
        }
      }
    }
  }
  if (!SPLIT && warp >= 6 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  if (SPLIT && warp < 6) {   // the epilogue warps' two cluster barriers, joined by all
    namespace cg = cooperative_groups;
    cg::this_cluster().sync();
    cg::this_cluster().sync();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(T_TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host: tensor maps ---------
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiled>(f);
  }();
  return fn;
}

// 5-D fp32 map; box = {box0, box1, 1, 1, 1}; swizzle128: 128-B swizzle (box0 = 32)
cudaError_t make_map(CUtensorMap* map, const float* base, const Tf32Dim& d, int box0, int box1, bool swizzle128) {
  EncodeTiled enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5] = {(cuuint32_t)box0, (cuuint32_t)box1, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) dims[i] = (cuuint64_t)(d.ext[i] < 1 ? 1 : d.ext[i]);
  long long prev = 1;   // element stride of dim i-1
  for (int i = 1; i < 5; ++i) {
    long long s = d.stride[i];
    // extent-1 dims are never stepped: give them the packed stride so every stride is a
    // multiple of 16 B whatever the caller wrote there
    if (dims[i] == 1 || s <= 0) s = prev * (long long)dims[i - 1];
    strides[i - 1] = (cuuint64_t)s * 4;
    if (strides[i - 1] % 16 || strides[i - 1] >= (1ULL << 40)) return cudaErrorInvalidValue;
    prev = s;
  }
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int num_sms_tf32() {
  static int nsm[32] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (nsm[dev] == 0 && (cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
                        nsm[dev] <= 0))
    nsm[dev] = 148;
  return nsm[dev];
}

}  // namespace

cudaError_t tf32_prepare() {
  static bool done[32] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) dev = 0;
  if (done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(tf32x3_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, T_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(tf32x3_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, T_SMEM);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

double tf32_gemm_flops(const Tf32Gemm& g) {
  return 2.0 * g.M * (double)g.N * (double)g.kseg * g.nseg * g.ns * g.nt * g.nb;
}

cudaError_t launch_tf32_gemm(const Tf32Gemm& g, cudaStream_t stream) {
  if (g.M <= 0 || g.N <= 0 || g.ns * g.nt * g.nb <= 0) return cudaSuccess;
  if (g.kseg <= 0 || g.nseg <= 0 || (g.kind == TF32_ROW && g.slo > 0 && g.nseg % g.slo != 0))
    return cudaErrorInvalidValue;
  cudaError_t e = tf32_prepare();
  if (e != cudaSuccess) return e;
  Tf32GemmArgs p;
  p.kind = g.kind;
  p.M = g.M;
  p.N = g.N;
  p.kseg = g.kseg;
  p.nseg = g.nseg;
  p.slo = g.slo < 1 ? 1 : g.slo;
  p.ns = g.ns;
  p.nt = g.nt;
  p.nb = g.nb;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.ldc = g.ldc;
  p.ldd = g.ldd;
  p.sC_t = g.sC_t;
  p.sC_b = g.sC_b;
  p.sD_t = g.sD_t;
  p.sD_b = g.sD_b;
  bool vec4 = g.N % 4 == 0 && g.ldc % 4 == 0 && g.ldd % 4 == 0 && g.sC_t % 4 == 0 && g.sC_b % 4 == 0 &&
              g.sD_t % 4 == 0 && g.sD_b % 4 == 0;
  for (int s = 0; s < MAXS; ++s) {
    p.C[s] = g.C[s];
    p.D[s] = g.beta != 0.0f ? g.D[s] : nullptr;
    for (const void* q : {(const void*)g.C[s], (const void*)p.D[s]})
      vec4 = vec4 && (reinterpret_cast<uintptr_t>(q) & 15) == 0;
  }
  p.vec4 = vec4;
  static const int nostore = getenv("KX_TF32_NOSTORE") ? 1 : 0;
  p.diag_nostore = nostore;
  static const bool no_tma_store = getenv("KX_TF32_ROWSTORE") != nullptr;   // A/B experiments only
  p.tma_store = 0;
  if (!no_tma_store) {
    bool ok = true;
    for (int s = 0; s < g.ns && ok; ++s) {
      Tf32Dim dc;
      dc.hi = g.C[s];
      dc.ext[0] = g.N, dc.ext[1] = g.M, dc.ext[2] = g.nt, dc.ext[3] = g.nb;
      dc.stride[1] = g.ldc, dc.stride[2] = g.sC_t, dc.stride[3] = g.sC_b;
      ok = (reinterpret_cast<uintptr_t>(g.C[s]) & 15) == 0 && make_map(&p.mapC[s], g.C[s], dc, 32, 32, true) == cudaSuccess;
    }
    p.tma_store = ok && vec4 ? 1 : 0;
    // in place with beta = 1 (U = U + ..., the last stage): the TMA unit adds the boxes into C,
    // so D is never loaded; same single round-to-nearest add as alpha acc + D
    static const bool no_reduce = getenv("KX_TF32_NOREDUCE") != nullptr;   // A/B experiments only
    bool inplace = p.tma_store && g.beta == 1.0f && !no_reduce && g.ldd == g.ldc && g.sD_t == g.sC_t && g.sD_b == g.sC_b;
    for (int s = 0; s < g.ns && inplace; ++s) inplace = g.D[s] == g.C[s];
    if (inplace) p.tma_store = 2;
  }
  const int mS = g.kind == TF32_COL ? TBM : TBN;   // static operand rows per tile
  if ((e = make_map(&p.mapS_hi, g.S.hi, g.S, TBK, mS, true)) != cudaSuccess) return e;
  if ((e = make_map(&p.mapS_lo, g.S.lo, g.S, TBK, mS, true)) != cudaSuccess) return e;
  if (g.kind == TF32_COL) e = make_map(&p.mapT, g.T.hi, g.T, TBN, TBK, false);   // raw [k][n]
  else e = make_map(&p.mapT, g.T.hi, g.T, TBK, TBM, true);                      // raw K-major
  if (e != cudaSuccess) return e;
  const long long tiles = (long long)((g.M + TBM - 1) / TBM) * ((g.N + TBN - 1) / TBN) * g.ns * g.nt * g.nb;
  const int nsm = num_sms_tf32();
  const int ktiles = (g.kseg + TBK - 1) / TBK * g.nseg;
  static const bool no_split = getenv("KX_TF32_NOSPLIT") != nullptr;   // diagnostics only
  static const bool trace = getenv("KX_TRACE") != nullptr;            // diagnostics only
  // cluster split-K factor for `t` tiles sharing the SMs (2, 4, 8; 0 = none)
  auto split_of = [&](long long t, int min_kt) {   // >= min_kt k-tiles per split CTA
    if (no_split || t * 2 > nsm || ktiles < 2 * min_kt) return 0;
    int S = 8;
    while (S > 1 && (t * S > nsm || ktiles < min_kt * S)) S /= 2;
    return S >= 2 ? S : 0;
  };
  auto launch_split = [&](long long t0, long long t1, int S) -> bool {
    p.csplit = S;
    p.tile0 = (int)t0;
    p.tile1 = (int)t1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((t1 - t0) * S));
    cfg.blockDim = dim3(T_THREADS);
    cfg.dynamicSmemBytes = T_SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tf32x3_gemm_kernel<true>, p) == cudaSuccess) return true;
    cudaGetLastError();   // refused (cluster residency)
    return false;
  };
  auto launch_persistent = [&](long long t0, long long t1) {
    p.csplit = 0;
    p.tile0 = (int)t0;
    p.tile1 = (int)t1;
    tf32x3_gemm_kernel<false><<<(int)std::min<long long>(t1 - t0, nsm), T_THREADS, T_SMEM, stream>>>(p);
    return cudaGetLastError();
  };
  // few tiles (small grids: the stage GEMMs of a 300^2 step have 18): every tile split over a
  // cluster; many tiles with a short last wave (768 = 5 x 148 + 28 at C2): the whole waves
  // persistent, then the tail tiles split over clusters (an S-times shorter last wave)
  // (the tail split pays only with >= 8 k-tiles per split CTA: at K = 128 (C3) it cost 12%)
  const int S_all = split_of(tiles, 2);
  const long long tail = tiles > nsm ? tiles % nsm : 0;
  const int S_tail = tail ? split_of(tail, 8) : 0;
  if (trace)
    fprintf(stderr, "kx-tf32 %s M=%d N=%d K=%dx%d z=%dx%dx%d tiles=%lld split=%d tail=%lld split_tail=%d\n",
            g.kind == TF32_COL ? "col" : "row", g.M, g.N, g.kseg, g.nseg, g.ns, g.nt, g.nb, tiles, S_all, tail,
            S_tail);
  if (S_all && launch_split(0, tiles, S_all)) return cudaSuccess;
  if (S_tail) {
    e = launch_persistent(0, tiles - tail);
    if (e != cudaSuccess) return e;
    if (launch_split(tiles - tail, tiles, S_tail)) return cudaSuccess;
    return launch_persistent(tiles - tail, tiles);
  }
  return launch_persistent(0, tiles);
}

}  // namespace kx
