// Probe of the tcgen05 building blocks the fp32 GEMM (csrc/tf32gemm.cu) relies on, one CTA:
//   T1  TMEM store / load round trip (lane/column addressing of tcgen05.st / tcgen05.ld)
//   T2  one kind::tf32 MMA (M = N = 128, K = 32 as 4 x K8), A K-major SW128, B K-major SW128
//   T3  the same with B MN-major SW128 (the layout the GEMM uses), LBO = 4096, SBO = 1024
// Operands are written into shared memory by the threads in the swizzled layout (no TMA).
// Prints max |error| against the exact products (small integers, exact in tf32).  Not a test.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(unsigned saddr, unsigned lbo, unsigned sbo, unsigned layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// swizzled byte offset of element e (< 32 floats) of 128-B row r
__device__ __forceinline__ unsigned sw128(unsigned r, unsigned e) {
  return r * 128 + ((((e >> 2) ^ (r & 7))) << 4) + (e & 3) * 4;
}

__global__ void probe(int test, float* out, unsigned bmajor) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;            // 128 x 32 floats = 16 KB
  uint8_t* sB = smem + 16384;    // 128 x 32 floats = 16 KB
  __shared__ uint64_t bar;
  __shared__ unsigned slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // A(m, k) = (m % 4) + 1 if k == m % 32 else 0 ... use a simple full pattern:
  //   A(m, k) = ((m + k) % 3) - 1,  B(k, n) = ((k * 7 + n) % 5) - 2
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int m = i / 32, k = i % 32;
    *(float*)(sA + (m / 8) * 1024 + sw128(m % 8, k)) = (float)(((m + k) % 3) - 1);
  }
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int n = i / 32, k = i % 32;
    const float v = (float)(((k * 7 + n) % 5) - 2);
    if (bmajor == 0) {   // K-major: row n (32 k), 8-row atoms of 1 KB
      *(float*)(sB + (n / 8) * 1024 + sw128(n % 8, k)) = v;
    } else {             // MN-major: 32-wide n chunks of 4 KB; row k (32 n)
      *(float*)(sB + (n / 32) * 4096 + (k / 8) * 1024 + sw128(k % 8, n % 32)) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const unsigned tmem = slot;
  if (test == 1) {
    // each warp stores lane*1000 + col into its lane quarter, 32 columns
    unsigned v[4];
    for (int j = 0; j < 4; ++j) v[j] = __float_as_uint((float)((warp * 32 + lane) * 1000 + j));
    const unsigned ta = tmem + ((unsigned)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(ta), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    unsigned r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int j = 0; j < 4; ++j) out[(warp * 32 + lane) * 128 + j] = __uint_as_float(r[j]);
  } else {
    if (warp == 0 && lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (bmajor << 16) |
                             ((128u >> 3) << 17) | ((128u >> 4) << 24);
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t dA = sdesc(su32(sA) + ks * 32, 16, 1024, 2);
        const uint64_t dB = bmajor ? sdesc(su32(sB) + ks * 1024, 4096, 1024, 2) : sdesc(su32(sB) + ks * 32, 16, 1024, 2);
        const unsigned acc = ks > 0;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(dA), "l"(dB), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                   : "memory");
    }
    __syncwarp();
    asm volatile(
        "{\n .reg .pred P1;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n" ::"r"(
            su32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    for (int cb = 0; cb < 128; cb += 8) {
      unsigned r[8];
      const unsigned ta = tmem + ((unsigned)(warp * 32) << 16) + cb;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) out[(warp * 32 + lane) * 128 + cb + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 128 * 4);
  float* h = new float[128 * 128];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int test = 1; test <= 3; ++test) {
    cudaMemset(d, 0, 128 * 128 * 4);
    probe<<<1, 128, 40 * 1024>>>(test == 1 ? 1 : 2, d, test == 3 ? 1u : 0u);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("T%d: CUDA error %s\n", test, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < (test == 1 ? 4 : 128); ++n) {
        double ref;
        if (test == 1) ref = m * 1000 + n;
        else {
          ref = 0;
          for (int k = 0; k < 32; ++k) ref += (double)(((m + k) % 3) - 1) * (double)(((k * 7 + n) % 5) - 2);
        }
        const double err = fabs(h[m * 128 + n] - ref);
        if (err > 0 && bad < 4) printf("  T%d (%d,%d) got %g want %g\n", test, m, n, h[m * 128 + n], ref);
        bad += err > 0;
        maxerr = err > maxerr ? err : maxerr;
        maxref = fabs(ref) > maxref ? fabs(ref) : maxref;
      }
    printf("T%d: max err %g (max |ref| %g), %d wrong\n", test, maxerr, maxref, bad);
  }
  return 0;
}
