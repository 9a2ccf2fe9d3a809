// fp32 mu-mode product GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32) with the
// three-pass split that recovers fp32 accuracy — the precision variant behind the paper's "CUDA
// single" columns (Table 5, Table 7).
//
// Every fp32 operand x is carried as two tf32-valued planes, hi = rna_tf32(x) and
// lo = rna_tf32(x - hi) (|x - hi - lo| <= 2^-22 |x|), produced by whoever writes the operand
// (this kernel's epilogue, the fp32 pointwise kernels, the bank conversion).  A product is then
//     A B ~ A_lo B_hi + A_hi B_lo + A_hi B_hi          (3 tf32 MMAs, fp32 accumulate in TMEM)
// which drops only the A_lo B_lo term (~2^-22 relative).  The mode products need no permutes
// (P:219-231): the A operand (the phi-matrix stack for mu >= 2, the tensor rows X_r for mu = 1)
// is K-major and the B operand (the tensor slab X_b for mu >= 2, L^T for mu = 1) is MN-major;
// tcgen05 reads both directly from 128-B-swizzled shared memory.
//
// Structure (one CTA per SM, persistent over output tiles of 128 x 128):
//   warp 0      TMA producer: per k-tile, 2 loads of A (hi, lo: 128 rows x 32 k) and 8 of B
//               (hi, lo: 4 chunks of 32 n x 32 k), completion counted on the stage's mbarrier;
//   warp 1      MMA issuer (one elected thread): 4 k-steps x 3 MMAs (M=128, N=128, K=8) per
//               k-tile into a double-buffered TMEM accumulator (2 x 128 columns); tcgen05.commit
//               frees the smem stage and, after the last k-tile, hands the accumulator over;
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 columns per warp, C = alpha acc + beta D,
//               stored as fp32 and/or as the (hi, lo) planes the next GEMM reads.
#include "kx_internal.h"

#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace kx {
namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3;
constexpr int T_A_BYTES = TBM * TBK * 4;          // 16 KB per plane
constexpr int T_B_BYTES = TBN * TBK * 4;          // 16 KB per plane
constexpr int T_STAGE_BYTES = 2 * (T_A_BYTES + T_B_BYTES);
constexpr int T_SMEM = TSTAGES * T_STAGE_BYTES + 1024 /* alignment */ + 256 /* barriers */;
constexpr int T_THREADS = 192;
constexpr int T_TMEM_COLS = 256;                  // 2 accumulators of 128 fp32 columns

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

// shared-memory matrix descriptor (tcgen05): start, leading / stride byte offsets (16-B units),
// version 1 (sm_100), 128-B swizzle
__device__ __forceinline__ uint64_t sdesc(unsigned saddr, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::tf32, fp32 accumulate, A K-major, B MN-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4)           // c_format F32
                            | (2u << 7)         // a_format TF32
                            | (2u << 10)        // b_format TF32
                            | (0u << 15)        // a_major K
                            | (1u << 16)        // b_major MN
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

struct Tf32GemmArgs {
  CUtensorMap mapA_hi, mapA_lo, mapB_hi, mapB_lo;   // 64-B aligned members first
  int kind, M, N, kseg, nseg, ns, nt, nb, vec4;
  float alpha, beta;
  long long ldc, ldd, sC_t, sC_b, sD_t, sD_b;
  float* C[MAXS];
  float* Ch[MAXS];
  float* Cl[MAXS];
  const float* D[MAXS];
};

struct TileCoord {
  int m0, n0, s, t, b;
};

__device__ __forceinline__ TileCoord tile_coord(const Tf32GemmArgs& p, int tiles_m, int tiles_n, int tl) {
  const int tmn = tiles_m * tiles_n;
  const int z = tl / tmn, r = tl - z * tmn;
  TileCoord c;
  if (p.kind == TF32_COL) {   // m fastest: consecutive CTAs share the big B panel
    c.m0 = (r % tiles_m) * TBM;
    c.n0 = (r / tiles_m) * TBN;
  } else {                    // n fastest: consecutive CTAs share the big A panel
    c.n0 = (r % tiles_n) * TBN;
    c.m0 = (r / tiles_n) * TBM;
  }
  c.b = z % p.nb;
  const int zt = z / p.nb;
  c.t = zt % p.nt;
  c.s = zt / p.nt;
  return c;
}

__global__ void __launch_bounds__(T_THREADS, 1) tf32x3_gemm_kernel(const __grid_constant__ Tf32GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TSTAGES * T_STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  uint64_t* tfull = empty + TSTAGES;    // accumulator ready (MMA -> epilogue), 2 buffers
  uint64_t* tempty = tfull + 2;         // accumulator drained (epilogue -> MMA)
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (p.M + TBM - 1) / TBM, tiles_n = (p.N + TBN - 1) / TBN;
  const int ntiles = tiles_m * tiles_n * p.ns * p.nt * p.nb;
  const int kps = (p.kseg + TBK - 1) / TBK;
  const int ktiles = kps * p.nseg;

  if (threadIdx.x == 0) {
    for (int i = 0; i < TSTAGES; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, 128);
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
      for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        const TileCoord c = tile_coord(p, tiles_m, tiles_n, tl);
        for (int kt = 0; kt < ktiles; ++kt, ++it) {
          const int st = it % TSTAGES, fill = it / TSTAGES;
          if (fill > 0) mbar_wait(empty + st, (fill - 1) & 1);
          uint8_t* sA = smem + st * T_STAGE_BYTES;
          uint8_t* sAl = sA + T_A_BYTES;
          uint8_t* sB = sAl + T_A_BYTES;
          uint8_t* sBl = sB + T_B_BYTES;
          mbar_expect_tx(full + st, T_STAGE_BYTES);
          const int seg = kt / kps, k0 = (kt - seg * kps) * TBK;
          int a2, a3, b1, b2, b3, b4;
          if (p.kind == TF32_COL) {
            a2 = c.t; a3 = c.s;                 // A: (k, m, t, s)
            b1 = k0; b2 = c.b; b3 = c.t; b4 = c.s;   // B: (n, k, b, t, s)
          } else {
            a2 = seg; a3 = c.s;                 // A: (k, m, seg, s)
            b1 = seg * p.kseg + k0; b2 = c.s; b3 = 0; b4 = 0;   // B: (n, kglob, s)
          }
          tma_load5(sA, &p.mapA_hi, k0, c.m0, a2, a3, 0, full + st);
          tma_load5(sAl, &p.mapA_lo, k0, c.m0, a2, a3, 0, full + st);
#pragma unroll
          for (int j = 0; j < TBN / 32; ++j) {
            tma_load5(sB + j * 4096, &p.mapB_hi, c.n0 + 32 * j, b1, b2, b3, b4, full + st);
            tma_load5(sBl + j * 4096, &p.mapB_lo, c.n0 + 32 * j, b1, b2, b3, b4, full + st);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int it = 0, tcount = 0;
    for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++tcount) {
      const int buf = tcount & 1, use = tcount >> 1;
      if (use > 0) mbar_wait(tempty + buf, (use - 1) & 1);   // epilogue drained this buffer
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const unsigned tmem_d = tmem_base + buf * TBN;
      for (int kt = 0; kt < ktiles; ++kt, ++it) {
        const int st = it % TSTAGES;
        mbar_wait(full + st, (it / TSTAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const unsigned a = su32(smem + st * T_STAGE_BYTES);
          const unsigned al = a + T_A_BYTES, b = al + T_A_BYTES, bl = b + T_B_BYTES;
#pragma unroll
          for (int ks = 0; ks < TBK / 8; ++ks) {
            // A K-major: k-step = 32 B inside the 128-B swizzled row; 8-row groups 1 KB apart
            // B MN-major: k-step = one 8-row (1 KB) group; 32-wide n chunks 4 KB apart
            const uint64_t dA = sdesc(a + ks * 32, 16, 1024), dAl = sdesc(al + ks * 32, 16, 1024);
            const uint64_t dB = sdesc(b + ks * 1024, 4096, 1024), dBl = sdesc(bl + ks * 1024, 4096, 1024);
            const unsigned acc0 = (kt > 0 || ks > 0) ? 1u : 0u;
            mma_tf32(tmem_d, dAl, dB, acc0);
            mma_tf32(tmem_d, dA, dBl, 1u);
            mma_tf32(tmem_d, dA, dB, 1u);
          }
          mma_commit(empty + st);                   // smem stage free once these MMAs finish
          if (kt == ktiles - 1) mma_commit(tfull + buf);   // accumulator complete
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    int tcount = 0;
    for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++tcount) {
      const TileCoord c = tile_coord(p, tiles_m, tiles_n, tl);
      const int buf = tcount & 1, use = tcount >> 1;
      mbar_wait(tfull + buf, use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int m = c.m0 + q * 32 + lane;
      const long long zoff_c = c.t * p.sC_t + c.b * p.sC_b;
      const long long zoff_d = c.t * p.sD_t + c.b * p.sD_b;
      float* C = p.C[c.s];
      float* Ch = p.Ch[c.s];
      float* Cl = p.Cl[c.s];
      const float* D = p.D[c.s];
      for (int cb = 0; cb < TBN; cb += 32) {
        unsigned v[32];
        const unsigned taddr = tmem_base + ((unsigned)(q * 32) << 16) + buf * TBN + cb;
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
        if (cb + 32 >= TBN) {   // whole accumulator read: hand the buffer back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          mbar_arrive(tempty + buf);
        }
        if (m >= p.M) continue;
        const int n0 = c.n0 + cb;
        const long long oc = zoff_c + (long long)m * p.ldc + n0;
        const long long od = zoff_d + (long long)m * p.ldd + n0;
        const bool full_row = n0 + 32 <= p.N && p.vec4;
        if (full_row) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 r = make_float4(p.alpha * __uint_as_float(v[j]), p.alpha * __uint_as_float(v[j + 1]),
                                   p.alpha * __uint_as_float(v[j + 2]), p.alpha * __uint_as_float(v[j + 3]));
            if (D) {
              const float4 dd = *reinterpret_cast<const float4*>(D + od + j);
              r.x += p.beta * dd.x;
              r.y += p.beta * dd.y;
              r.z += p.beta * dd.z;
              r.w += p.beta * dd.w;
            }
            if (C) *reinterpret_cast<float4*>(C + oc + j) = r;
            if (Ch) {
              const float4 h = make_float4(tf32_rna(r.x), tf32_rna(r.y), tf32_rna(r.z), tf32_rna(r.w));
              *reinterpret_cast<float4*>(Ch + oc + j) = h;
              *reinterpret_cast<float4*>(Cl + oc + j) =
                  make_float4(tf32_rna(r.x - h.x), tf32_rna(r.y - h.y), tf32_rna(r.z - h.z), tf32_rna(r.w - h.w));
            }
          }
        } else {
          for (int j = 0; j < 32 && n0 + j < p.N; ++j) {
            float r = p.alpha * __uint_as_float(v[j]);
            if (D) r += p.beta * D[od + j];
            if (C) C[oc + j] = r;
            if (Ch) {
              const float h = tf32_rna(r);
              Ch[oc + j] = h;
              Cl[oc + j] = tf32_rna(r - h);
            }
          }
        }
      }
    }
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

// 5-D fp32 map with a 128-B swizzle; box = {32, box1, 1, 1, 1}
cudaError_t make_map(CUtensorMap* map, const float* base, const Tf32Dim& d, int box1) {
  EncodeTiled enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5] = {32, (cuuint32_t)box1, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) dims[i] = (cuuint64_t)(d.ext[i] < 1 ? 1 : d.ext[i]);
  for (int i = 1; i < 5; ++i) {
    long long s = d.stride[i];
    if (s <= 0) s = d.stride[i - 1] * (long long)dims[i - 1];   // unused extent-1 dims
    if (s <= 0) s = 1;
    strides[i - 1] = (cuuint64_t)s * 4;
    if (strides[i - 1] % 16) return cudaErrorInvalidValue;
  }
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
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
  cudaError_t e = cudaFuncSetAttribute(tf32x3_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, T_SMEM);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

double tf32_gemm_flops(const Tf32Gemm& g) {
  return 2.0 * g.M * (double)g.N * (double)g.kseg * g.nseg * g.ns * g.nt * g.nb;
}

cudaError_t launch_tf32_gemm(const Tf32Gemm& g, cudaStream_t stream) {
  if (g.M <= 0 || g.N <= 0 || g.ns * g.nt * g.nb <= 0) return cudaSuccess;
  if (g.kseg <= 0 || g.nseg <= 0) return cudaErrorInvalidValue;
  cudaError_t e = tf32_prepare();
  if (e != cudaSuccess) return e;
  Tf32GemmArgs p;
  p.kind = g.kind;
  p.M = g.M;
  p.N = g.N;
  p.kseg = g.kseg;
  p.nseg = g.nseg;
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
    p.Ch[s] = g.Ch[s];
    p.Cl[s] = g.Cl[s];
    p.D[s] = g.beta != 0.0f ? g.D[s] : nullptr;
    for (const void* q : {(const void*)g.C[s], (const void*)g.Ch[s], (const void*)g.Cl[s], (const void*)p.D[s]})
      vec4 = vec4 && (reinterpret_cast<uintptr_t>(q) & 15) == 0;
  }
  p.vec4 = vec4;
  if ((e = make_map(&p.mapA_hi, g.A.hi, g.A, TBM)) != cudaSuccess) return e;
  if ((e = make_map(&p.mapA_lo, g.A.lo, g.A, TBM)) != cudaSuccess) return e;
  if ((e = make_map(&p.mapB_hi, g.B.hi, g.B, TBK)) != cudaSuccess) return e;
  if ((e = make_map(&p.mapB_lo, g.B.lo, g.B, TBK)) != cudaSuccess) return e;
  const long long tiles = (long long)((g.M + TBM - 1) / TBM) * ((g.N + TBN - 1) / TBN) * g.ns * g.nt * g.nb;
  const int grid = (int)std::min<long long>(tiles, num_sms_tf32());
  static const bool trace = getenv("KX_TRACE") != nullptr;   // diagnostics only
  if (trace)
    fprintf(stderr, "kx-tf32 %s M=%d N=%d K=%dx%d z=%dx%dx%d tiles=%lld grid=%d\n",
            g.kind == TF32_COL ? "col" : "row", g.M, g.N, g.kseg, g.nseg, g.ns, g.nt, g.nb, tiles, grid);
  tf32x3_gemm_kernel<<<grid, T_THREADS, T_SMEM, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace kx
