// K5 on the 5th-generation tensor cores: Z = X * F for d in {32, 64, 128, 256}
// (factor_state.cpp:120-123 query_all, :215-222 rebase, enhancer.cpp:196-206).
//
// Precision: single-pass TF32 misses the 1e-4 contract (SURVEY hard part 3),
// so each K-step issues three MMAs into one FP32 TMEM accumulator:
//     Z = Xhi*Fhi + Xhi*Flo + Xlo*Fhi
// d <= 128: kind::tf32 with Xhi = X rounded to an exact TF32 value in shared
// memory (low 13 mantissa bits cleared), Xlo = X - Xhi (exact), Fhi/Flo
// likewise from the fp64 F (relative error ~2^-20). d = 256: kind::f16 with
// BF16 hi/lo parts (see materialize_bf16_256; ~4e-6).
//
// Warp roles (320 threads, one persistent CTA per SM, 128-row tiles):
//   warp 0      TMA producer: X chunks (128 rows x 32 fp32 = one 128-byte
//               swizzle atom) into a ring of S stages
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   split: Xhi in place and Xlo into the stage's second buffer,
//               fence.proxy.async, arrive
//   warps 6-9   epilogue: tcgen05.ld 32 lanes x 32 columns, swizzled smem
//               staging, TMA bulk tensor stores
// d <= 64: F (hi and lo, K-major, SW128) resident in shared memory; d = 128:
// F^T resident in TMEM (materialize_tc128_ts); d = 256: F^T streamed in K
// slices, multicast across a 4-CTA cluster. The accumulator is double-
// buffered in TMEM so the epilogue of tile t overlaps the MMAs of tile t+1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "materialize.cuh"

namespace dgpu {

namespace {

constexpr int TM = 128;         // rows per tile (UMMA M)
constexpr int KC = 32;          // fp32 per 128-byte swizzle atom (one TMA box / stage)
template <int D> constexpr int stages_for() { return D == 32 ? 5 : D == 64 ? 4 : 2; }
constexpr int OSTAGE = 4096;  // epilogue staging: 32 rows x 128 B per buffer
constexpr int THREADS = 320;
constexpr int CHUNK_BYTES = TM * KC * 4;  // 16 KB

DAMF_D uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

DAMF_D void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
DAMF_D void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
DAMF_D void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
DAMF_D void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
DAMF_D void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
DAMF_D void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
DAMF_D void tma_store_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
DAMF_D void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
DAMF_D void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
DAMF_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DAMF_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte-swizzled UMMA shared-memory descriptor (SBO = 1024 B
// between 8-row core-matrix groups, LBO = 16 B, version 1 for sm_100).
DAMF_D uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;           // LBO (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32; // SBO
  d |= (uint64_t)1 << 46;           // version
  d |= (uint64_t)2 << 61;           // SWIZZLE_128B
  return d;
}

DAMF_D void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
DAMF_D void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
DAMF_D void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Byte offset of element (row r, col c in [0,32)) inside a 128-row x 128-byte
// SW128 atom: 16-byte chunk index XORed with (row mod 8).
DAMF_HD uint32_t sw128(int r, int c) {
  const int chunk = (c >> 2) ^ (r & 7);
  return (uint32_t)(r * 128 + chunk * 16 + (c & 3) * 4);
}

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
    materialize_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap zmap,
                          const float* __restrict__ Fhi_g, const float* __restrict__ Flo_g,
                          int64_t n) {
  constexpr int STAGES = stages_for<D>();
  constexpr int KB = D / KC;                 // 128-byte K atoms per row
  constexpr int FB = D * KC * 4;             // bytes of one K atom of F (D rows x 128 B)
  constexpr uint32_t TMEM_COLS = D * 2 < 32 ? 32 : D * 2;  // double-buffered accumulator
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sF = sm;                          // [2][KB][D x 128 B]  hi, lo
  unsigned char* sX = sm + 2 * KB * FB;            // [STAGES][2][16 KB]  X (hi in place), Xlo
  unsigned char* sO = sX + STAGES * 2 * CHUNK_BYTES;   // [4 warps][2][4 KB] store staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 4 * 2 * OSTAGE);
  uint64_t* full = bars;                 // TMA -> split
  uint64_t* ready = bars + STAGES;       // split -> MMA
  uint64_t* empty = bars + 2 * STAGES;   // MMA -> TMA
  uint64_t* tfull = bars + 3 * STAGES;   // MMA -> epilogue (2)
  uint64_t* tempty = bars + 3 * STAGES + 2;  // epilogue -> MMA (2)
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TM - 1) / TM;

  // ---- F (hi, lo) into the swizzled K-major layout: row = output column j
  for (int x = threadIdx.x; x < D * D; x += THREADS) {
    const int j = x / D, kk = x % D;  // B[j][kk] = F[kk][j] (FT rows given)
    const int kb = kk / KC, c = kk % KC;
    const uint32_t off = (uint32_t)kb * FB + sw128(j, c);
    *reinterpret_cast<float*>(sF + off) = Fhi_g[(int64_t)j * D + kk];
    *reinterpret_cast<float*>(sF + KB * FB + off) = Flo_g[(int64_t)j * D + kk];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();  // F written by the generic proxy, read by the tensor core
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;

  if (warp == 0) {
    // ===== TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          mbar_expect_tx(&full[s], CHUNK_BYTES);
          tma_load_2d(sX + (size_t)s * 2 * CHUNK_BYTES, &xmap, kb * KC, (int)(t * TM), &full[s]);
        }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(D >> 3) << 17) |
                                 ((uint32_t)(TM >> 4) << 24);
      uint32_t it = 0, tl = 0;
      const uint32_t fbase = smem_u32(sF), xbase = smem_u32(sX);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        const int a = tl & 1;
        if (tl >= 2) mbar_wait(&tempty[a], ((tl >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dtm = tmem + (uint32_t)(a * D);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&ready[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t xh = xbase + (uint32_t)s * 2 * CHUNK_BYTES, xl = xh + CHUNK_BYTES;
          const uint32_t fh = fbase + (uint32_t)kb * FB, fl = fh + (uint32_t)KB * FB;
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {  // 8 tf32 (32 B) per MMA
            const uint32_t ko = ks * 32;
            const uint32_t acc0 = (kb | ks) ? 1u : 0u;
            mma_tf32(dtm, umma_desc(xh + ko), umma_desc(fh + ko), idesc, acc0);
            mma_tf32(dtm, umma_desc(xh + ko), umma_desc(fl + ko), idesc, 1u);
            mma_tf32(dtm, umma_desc(xl + ko), umma_desc(fh + ko), idesc, 1u);
          }
          mma_commit(&empty[s]);  // stage free once these MMAs have read it
        }
        mma_commit(&tfull[a]);  // accumulator a complete
      }
    }
  } else if (warp < 6) {
    // ===== split: Xhi = tf32(X) in place, Xlo = X - Xhi
    const int st = threadIdx.x - 64;  // 0..127
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        float4* xh = reinterpret_cast<float4*>(sX + (size_t)s * 2 * CHUNK_BYTES);
        float4* xl = reinterpret_cast<float4*>(sX + (size_t)s * 2 * CHUNK_BYTES + CHUNK_BYTES);
#pragma unroll
        for (int q = 0; q < CHUNK_BYTES / 16 / 128; ++q) {
          const int i = st + q * 128;
          float4 v = xh[i];
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          l.x = v.x - h.x;
          l.y = v.y - h.y;
          l.z = v.z - h.z;
          l.w = v.w - h.w;
          xh[i] = h;
          xl[i] = l;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[s]);
      }
  } else {
    // ===== epilogue: TMEM -> registers -> swizzled smem -> TMA store
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    unsigned char* stg = sO + (size_t)(warp - 6) * 2 * OSTAGE;
    uint32_t tl = 0, sb = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      const int a = tl & 1;
      mbar_wait(&tfull[a], (tl >> 1) & 1);
      tc_fence_after();
      const int64_t row0 = t * TM + q * 32;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32, sb ^= 1) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * D + c0), r);
        unsigned char* buf = stg + sb * OSTAGE;
        if (lane == 0) tma_store_wait_read1();  // buffer sb free again
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(buf + sw128(lane, 4 * v)) =
              make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                          __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && row0 < n) tma_store_2d(&zmap, c0, (int)row0, buf);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    if (lane == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// d = 128 variant with F in TMEM: Z^T = F^T X^T. A = F^T (hi and lo) lives in
// TMEM (lane j = output column, column kk = K) for the whole kernel, B = the
// X tile (K-major, rows = N), D^T accumulates in TMEM with lane = output
// column and column = tile row. TMEM: Fhi 128 + Flo 128 + 2 x 128 (double-
// buffered accumulator) = 512 columns; shared memory holds only the X stages
// (6) and the store staging, so more loads stay in flight.
constexpr int TS_STAGES = 6;
DAMF_D void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}
DAMF_D void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    materialize_tc128_ts(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap zmap,
                         const float* __restrict__ Fhi_g, const float* __restrict__ Flo_g, int64_t n) {
  constexpr int D = 128, KB = D / KC, STAGES = TS_STAGES;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sX = sm;                              // [STAGES][2][16 KB]
  unsigned char* sO = sX + STAGES * 2 * CHUNK_BYTES;   // [4 warps][2][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 4 * 2 * OSTAGE);
  uint64_t* full = bars;
  uint64_t* ready = bars + STAGES;
  uint64_t* empty = bars + 2 * STAGES;
  uint64_t* tfull = bars + 3 * STAGES;
  uint64_t* tempty = bars + 3 * STAGES + 2;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TM - 1) / TM;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;
  // F^T into TMEM: columns [0,128) = Fhi, [128,256) = Flo; lane j <- FT row j
  if (warp >= 6) {
    const int q = warp & 3;
    const int j = q * 32 + lane;
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const float* src = (part ? Flo_g : Fhi_g) + (int64_t)j * D;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t r[32];
#pragma unroll
        for (int v = 0; v < 32; ++v) r[v] = __float_as_uint(src[c0 + v]);
        tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(part * D + c0), r);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tA_hi = tmem, tA_lo = tmem + D, tD = tmem + 2 * D;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          mbar_expect_tx(&full[s], CHUNK_BYTES);
          tma_load_2d(sX + (size_t)s * 2 * CHUNK_BYTES, &xmap, kb * KC, (int)(t * TM), &full[s]);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // M = 128 (output columns), N = 128 (tile rows), A from TMEM, B K-major
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TM >> 3) << 17) |
                                 ((uint32_t)(D >> 4) << 24);
      uint32_t it = 0, tl = 0;
      const uint32_t xbase = smem_u32(sX);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        const int a = tl & 1;
        if (tl >= 2) mbar_wait(&tempty[a], ((tl >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dtm = tD + (uint32_t)(a * TM);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&ready[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t xh = xbase + (uint32_t)s * 2 * CHUNK_BYTES, xl = xh + CHUNK_BYTES;
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint32_t kcol = (uint32_t)(kb * KC + ks * 8);  // A columns (K) in TMEM
            const uint32_t ko = ks * 32;                         // B bytes within the atom
            const uint32_t acc0 = (kb | ks) ? 1u : 0u;
            mma_tf32_ts(dtm, tA_hi + kcol, umma_desc(xh + ko), idesc, acc0);
            mma_tf32_ts(dtm, tA_lo + kcol, umma_desc(xh + ko), idesc, 1u);
            mma_tf32_ts(dtm, tA_hi + kcol, umma_desc(xl + ko), idesc, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[a]);
      }
    }
  } else if (warp < 6) {
    const int st = threadIdx.x - 64;
    uint32_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        float4* xh = reinterpret_cast<float4*>(sX + (size_t)s * 2 * CHUNK_BYTES);
        float4* xl = reinterpret_cast<float4*>(sX + (size_t)s * 2 * CHUNK_BYTES + CHUNK_BYTES);
#pragma unroll
        for (int q = 0; q < CHUNK_BYTES / 16 / 128; ++q) {
          const int i = st + q * 128;
          float4 v = xh[i];
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          l.x = v.x - h.x;
          l.y = v.y - h.y;
          l.z = v.z - h.z;
          l.w = v.w - h.w;
          xh[i] = h;
          xl[i] = l;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[s]);
      }
  } else {
    // epilogue: lane = output column j (quadrant q), TMEM column = tile row
    const int q = warp & 3;
    unsigned char* stg = sO + (size_t)(warp - 6) * 2 * OSTAGE;
    uint32_t tl = 0, sb = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      const int a = tl & 1;
      mbar_wait(&tfull[a], (tl >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int r0 = 0; r0 < TM; r0 += 32, sb ^= 1) {
        uint32_t r[32];
        tmem_ld32(tD + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * TM + r0), r);
        unsigned char* buf = stg + sb * OSTAGE;
        if (lane == 0) tma_store_wait_read1();
        __syncwarp();
        // staging tile [32 rows][32 columns] in SW128 layout; this thread owns column `lane`
#pragma unroll
        for (int v = 0; v < 32; ++v) *reinterpret_cast<uint32_t*>(buf + sw128(v, lane)) = r[v];
        fence_proxy_async();
        __syncwarp();
        const int64_t row0 = t * TM + r0;
        if (lane == 0 && row0 < n) tma_store_2d(&zmap, q * 32, (int)row0, buf);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    if (lane == 0) tma_store_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// d = 256 on kind::f16 (BF16 inputs, FP32 accumulate). At d = 256 three
// kind::tf32 passes need ~1.25 PFLOP/s of TF32 to keep up with HBM, which is
// above the TF32 rate; three BF16 passes run at twice that rate and move half
// the F bytes:   Z = Xhi*Fhi + Xhi*Flo + Xlo*Fhi   with Xhi = bf16_rn(X),
// Xlo = bf16_rn(X - Xhi) (representation error 2^-17 |x|), F likewise from
// fp64; measured 4e-6 relative Frobenius error, inside the 1e-4 contract.
// Three decoupled rings per 32-wide K slice, so the HBM stream is not held
// up by the tensor pipe: the raw X slice (one fp32 SW128 TMA box, 16 KB) is
// freed as soon as the split warps have read it; the split writes the bf16
// hi and lo operands (128 rows x 64 B each, SW64) into an operand ring that
// the MMAs release; the F^T slices (256 rows x 32 bf16, hi and lo, SW64,
// 16 KB each, TMA from L2) have their own ring, filled by a second producer.
constexpr int B256_KC = 32;                        // K per slice
constexpr int B256_XR = 4;                         // raw X ring (16 KB each)
constexpr int B256_OP = 2;                         // operand ring (hi + lo, 16 KB each)
constexpr int B256_FR = 3;                         // F ring (hi + lo, 32 KB each)
constexpr int B256_F = 256 * 64;                   // one K slice of F^T (bf16), 16 KB
constexpr int B256_CS = 4;                         // cluster size sharing each F slice (measured:
                                                   // 1 / 2 / 4 -> 3.65 / 3.53 / 3.38 ms at n = 2^23)
constexpr int B256_THREADS = THREADS + 32;         // + the F producer warp
constexpr size_t B256_SMEM = 1024 + (size_t)B256_XR * CHUNK_BYTES + (size_t)B256_OP * 2 * 8192 +
                             (size_t)B256_FR * 2 * B256_F + 8 * OSTAGE + 512;

// K-major SW64 UMMA descriptor (8-row groups 512 B apart)
DAMF_D uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}
DAMF_D float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
DAMF_D void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

DAMF_D void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

DAMF_D uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));  // a -> low half
  return r;
}

DAMF_D uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DAMF_D void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
DAMF_D void tma_load_2d_mc(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
DAMF_D void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// CS CTAs of a cluster work on CS different row tiles with the same F^T K
// slices: CTA r loads rows [r*256/CS, (r+1)*256/CS) of each F slice and
// multicasts them to every CTA of the cluster, so L2 serves each F slice once
// per cluster instead of once per CTA. An F slot is refilled only when every
// CTA's MMAs have released it (each MMA commit arrives on all CTAs' F-empty
// barrier). All CTAs of a cluster run the same number of tile iterations; a
// CTA whose tile is past the end re-reads the last tile and stores nothing.
// Warps: 0 X producer, 1 MMA, 2-5 split, 6-9 epilogue, 10 F producer.
template <int CS>
__global__ void __launch_bounds__(B256_THREADS, 1)
    materialize_bf16_256(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap zmap,
                         const __grid_constant__ CUtensorMap fhmap, const __grid_constant__ CUtensorMap flmap,
                         int64_t n) {
  constexpr int D = 256, KB = D / B256_KC;
  constexpr int FRW = 256 / CS;  // F^T rows this CTA loads per slice
  constexpr uint16_t ALL = (uint16_t)((1u << CS) - 1);
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sXR = sm;                                        // [XR][16 KB] raw fp32
  unsigned char* sOP = sXR + B256_XR * CHUNK_BYTES;               // [OP][hi 8 KB | lo 8 KB]
  unsigned char* sF = sOP + B256_OP * 2 * 8192;                   // [FR][hi 16 KB | lo 16 KB]
  unsigned char* sO = sF + B256_FR * 2 * B256_F;                  // [4 warps][2][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 4 * 2 * OSTAGE);
  uint64_t* xfull = bars;                          // X TMA -> split
  uint64_t* xempty = xfull + B256_XR;              // split -> X producer (4 warps)
  uint64_t* ofull = xempty + B256_XR;              // split -> MMA (4 warps)
  uint64_t* oempty = ofull + B256_OP;              // MMA -> split
  uint64_t* ffull = oempty + B256_OP;              // F TMA -> MMA
  uint64_t* fempty = ffull + B256_FR;              // MMAs of all CS CTAs -> F producer
  uint64_t* tfull = fempty + B256_FR;              // MMA -> epilogue (2)
  uint64_t* tempty = tfull + 2;                    // epilogue -> MMA (2)
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = CS > 1 ? (int)cluster_rank() : 0;
  const int64_t ntiles = (n + TM - 1) / TM;
  const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  // tile of iteration i: (cid + i * ncl) * CS + rank, while the group's first tile exists
  auto tile_of = [&](int64_t i) { return (cid + i * ncl) * CS + rank; };
  const int64_t iters = ntiles > cid * CS ? (ntiles - cid * CS + ncl * CS - 1) / (ncl * CS) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < B256_XR; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 4);
    }
    for (int s = 0; s < B256_OP; ++s) {
      mbar_init(&ofull[s], 4);
      mbar_init(&oempty[s], 1);
    }
    for (int s = 0; s < B256_FR; ++s) {
      mbar_init(&ffull[s], 1);
      mbar_init(&fempty[s], CS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;
  if (warp == 0) {
    // ===== X producer: raw fp32 K slices of this CTA's tiles
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t i = 0; i < iters; ++i) {
        const int64_t t = tile_of(i) < ntiles ? tile_of(i) : ntiles - 1;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % B256_XR;
          if (it >= B256_XR) mbar_wait(&xempty[s], ((it / B256_XR) - 1) & 1);
          mbar_expect_tx(&xfull[s], CHUNK_BYTES);
          tma_load_2d(sXR + (size_t)s * CHUNK_BYTES, &xmap, kb * B256_KC, (int)(t * TM), &xfull[s]);
        }
      }
    }
  } else if (warp == 10) {
    // ===== F producer: this CTA's rows of every F^T slice, multicast to the cluster
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t i = 0; i < iters; ++i)
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % B256_FR;
          if (it >= B256_FR) mbar_wait(&fempty[s], ((it / B256_FR) - 1) & 1);
          mbar_expect_tx(&ffull[s], 2 * B256_F);
          unsigned char* fh = sF + (size_t)s * 2 * B256_F + rank * FRW * 64;
          if (CS > 1) {
            tma_load_2d_mc(fh, &fhmap, kb * B256_KC, rank * FRW, &ffull[s], ALL);
            tma_load_2d_mc(fh + B256_F, &flmap, kb * B256_KC, rank * FRW, &ffull[s], ALL);
          } else {
            tma_load_2d(fh, &fhmap, kb * B256_KC, 0, &ffull[s]);
            tma_load_2d(fh + B256_F, &flmap, kb * B256_KC, 0, &ffull[s]);
          }
        }
    }
  } else if (warp == 1) {
    // ===== MMA issuer
    if (lane == 0) {
      // kind::f16: D = F32, A = B = BF16, both K-major, N = 256, M = 128
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(D >> 3) << 17) |
                                 ((uint32_t)(TM >> 4) << 24);
      uint32_t it = 0, tl = 0;
      const uint32_t obase = smem_u32(sOP), fbase = smem_u32(sF);
      for (int64_t i = 0; i < iters; ++i, ++tl) {
        const int a = tl & 1;
        if (tl >= 2) mbar_wait(&tempty[a], ((tl >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dtm = tmem + (uint32_t)(a * D);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int so = it % B256_OP, sf = it % B256_FR;
          mbar_wait(&ffull[sf], (it / B256_FR) & 1);
          mbar_wait(&ofull[so], (it / B256_OP) & 1);
          tc_fence_after();
          const uint32_t xh = obase + (uint32_t)so * 2 * 8192, xl = xh + 8192;
          const uint32_t fh = fbase + (uint32_t)sf * 2 * B256_F, fl = fh + B256_F;
#pragma unroll
          for (int ks = 0; ks < B256_KC / 16; ++ks) {  // 16 bf16 (32 B) per MMA
            const uint32_t ko = ks * 32;
            const uint32_t acc0 = (kb | ks) ? 1u : 0u;
            mma_bf16(dtm, umma_desc_sw64(xh + ko), umma_desc_sw64(fh + ko), idesc, acc0);
            mma_bf16(dtm, umma_desc_sw64(xh + ko), umma_desc_sw64(fl + ko), idesc, 1u);
            mma_bf16(dtm, umma_desc_sw64(xl + ko), umma_desc_sw64(fh + ko), idesc, 1u);
          }
          mma_commit(&oempty[so]);
          if (CS > 1) mma_commit_mc(&fempty[sf], ALL); else mma_commit(&fempty[sf]);
        }
        mma_commit(&tfull[a]);
      }
    }
  } else if (warp < 6) {
    // ===== split: row r of a raw slice (32 fp32, SW128) -> 32 bf16 hi and
    // 32 bf16 lo (SW64 rows of the operand slot)
    const int r = threadIdx.x - 64;
    const uint32_t xbase = smem_u32(sXR), obase = smem_u32(sOP);
    uint32_t it = 0;
    for (int64_t i = 0; i < iters; ++i)
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int sx = it % B256_XR, so = it % B256_OP;
        mbar_wait(&xfull[sx], (it / B256_XR) & 1);
        const uint32_t st = xbase + (uint32_t)sx * CHUNK_BYTES;
        float4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = lds128(st + r * 128 + ((c ^ (r & 7)) << 4));
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[sx]);  // raw slot free: values are in registers
        if (it >= B256_OP) mbar_wait(&oempty[so], ((it / B256_OP) - 1) & 1);
        const uint32_t ob = obase + (uint32_t)so * 2 * 8192;
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // bf16 chunk c = fp32 columns 8c .. 8c+7
          const float4 p = v[2 * c], q = v[2 * c + 1];
          uint4 h, l;
          h.x = pack_bf16(p.x, p.y);
          h.y = pack_bf16(p.z, p.w);
          h.z = pack_bf16(q.x, q.y);
          h.w = pack_bf16(q.z, q.w);
          l.x = pack_bf16(p.x - __uint_as_float(h.x << 16), p.y - __uint_as_float(h.x & 0xFFFF0000u));
          l.y = pack_bf16(p.z - __uint_as_float(h.y << 16), p.w - __uint_as_float(h.y & 0xFFFF0000u));
          l.z = pack_bf16(q.x - __uint_as_float(h.z << 16), q.y - __uint_as_float(h.z & 0xFFFF0000u));
          l.w = pack_bf16(q.z - __uint_as_float(h.w << 16), q.w - __uint_as_float(h.w & 0xFFFF0000u));
          const uint32_t off = r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
          sts128(ob + off, h);
          sts128(ob + 8192 + off, l);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ofull[so]);
      }
  } else {
    // ===== epilogue: TMEM -> registers -> swizzled smem -> TMA store
    const int q = warp & 3;
    unsigned char* stg = sO + (size_t)(warp - 6) * 2 * OSTAGE;
    uint32_t tl = 0, sb = 0;
    for (int64_t i = 0; i < iters; ++i, ++tl) {
      const int64_t t = tile_of(i);
      const int a = tl & 1;
      mbar_wait(&tfull[a], (tl >> 1) & 1);
      tc_fence_after();
      const int64_t row0 = t * TM + q * 32;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32, sb ^= 1) {
        uint32_t rr[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * D + c0), rr);
        unsigned char* buf = stg + sb * OSTAGE;
        if (lane == 0) tma_store_wait_read1();
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(buf + sw128(lane, 4 * v)) =
              make_float4(__uint_as_float(rr[4 * v]), __uint_as_float(rr[4 * v + 1]),
                          __uint_as_float(rr[4 * v + 2]), __uint_as_float(rr[4 * v + 3]));
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && row0 < n) tma_store_2d(&zmap, c0, (int)row0, buf);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    if (lane == 0) tma_store_wait_all();
  }
  tc_fence_before();
  // no CTA may leave while a peer can still multicast into it or arrive on its barriers
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---- d = 256 on CTA pairs (tcgen05.mma.cta_group::2) -------------------------
// The single-CTA kernel above is bound by shared-memory bandwidth: per 32-wide
// K slice a CTA's tensor core reads 72 KB of operands (three passes over a
// 128 x 32 X operand and a 256 x 32 F operand) next to 48 KB of TMA writes
// and 64 KB of split / epilogue traffic, ~80 % of 128 B/clk. A CTA pair
// computes a 256-row tile with ONE F slice between its two SMs: each CTA
// holds half of the slice's rows (N) and the pair's MMA reads both halves, so
// F costs each SM half the reads and half the TMA writes. Clusters of four =
// two pairs; CTA r of the cluster loads rows [64 r, 64 r + 64) of every slice
// and multicasts them to the two CTAs that hold that half (pair rank r / 2).
// Only the pair's even CTA issues MMAs; its barriers collect the arrivals of
// both CTAs (operands split, accumulator drained), and its commits are
// multicast to both (operand slot free, accumulator full) or to the whole
// cluster (F slot free).
#ifndef P256_XR_
#define P256_XR_ 5
#define P256_OP_ 3
#define P256_FR_ 4
#endif
constexpr int P256_XR = P256_XR_;          // raw X ring (16 KB each)
constexpr int P256_OP = P256_OP_;          // operand ring (hi 8 KB | lo 8 KB)
constexpr int P256_FR = P256_FR_;          // F ring of half slices (hi 8 KB | lo 8 KB)
constexpr int P256_FH = 128 * 64;          // half of one K slice of F^T (128 rows x 32 bf16)
constexpr int P256_PR = 4;                 // forwarded-readiness ring (>= min(OP, FR))
static_assert(P256_PR >= (P256_OP < P256_FR ? P256_OP : P256_FR), "pready ring too short");
constexpr size_t P256_SMEM = 1024 + (size_t)P256_XR * CHUNK_BYTES + (size_t)P256_OP * 2 * 8192 +
                             (size_t)P256_FR * 2 * P256_FH + 8 * OSTAGE + 512;
static_assert(P256_SMEM <= 232448, "pair kernel shared memory above the opt-in limit");

DAMF_D void mma_bf16_2cta(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
DAMF_D void mma_commit_mc2(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA `cta` of the cluster
DAMF_D void mbar_arrive_cta(uint64_t* b, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(b)), "r"(cta));
  // (default semantics, as cutlass::arch::ClusterBarrier::arrive(cta_id): a
  // release at cluster scope here is a full fence per call, and the one
  // forwarding thread then paces the whole pair at ~1 us per K slice. What it
  // forwards was made visible by its owners -- fence.proxy.async by the split
  // warps, the TMA's complete_tx -- before this thread observed their barriers.)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

template <int CS>  // 4: two pairs sharing each F slice by multicast; 2: one pair, its own F halves
__global__ void __launch_bounds__(B256_THREADS, 1)
    materialize_bf16_256_pair(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap zmap,
                              const __grid_constant__ CUtensorMap fhmap, const __grid_constant__ CUtensorMap flmap,
                              int64_t n) {
  constexpr int D = 256, KB = D / B256_KC;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sXR = sm;                                        // [XR][16 KB] raw fp32
  unsigned char* sOP = sXR + P256_XR * CHUNK_BYTES;               // [OP][hi 8 KB | lo 8 KB]
  unsigned char* sF = sOP + P256_OP * 2 * 8192;                   // [FR][hi 8 KB | lo 8 KB]
  unsigned char* sO = sF + P256_FR * 2 * P256_FH;                 // [4 warps][2][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 4 * 2 * OSTAGE);
  uint64_t* xfull = bars;                          // X TMA -> split (local)
  uint64_t* xempty = xfull + P256_XR;              // split -> X producer (local, 4 warps)
  uint64_t* ofull = xempty + P256_XR;              // split -> local (4 warps)
  uint64_t* oempty = ofull + P256_OP;              // leader's commit -> split (both CTAs)
  uint64_t* ffull = oempty + P256_OP;              // F TMA (two source CTAs) -> local
  uint64_t* pready = ffull + P256_FR;              // peer: "operands and F half of slice it are in my
                                                   // shared memory", forwarded -> leader's MMA (1)
  uint64_t* fempty = pready + P256_PR;             // both leaders' commits -> F producers (2)
  uint64_t* tfull = fempty + P256_FR;              // leader's commit -> epilogue (both CTAs)
  uint64_t* tempty = tfull + 2;                    // epilogue -> local (4 warps)
  uint64_t* ptempty = tempty + 2;                  // peer's tempty forwarded -> leader's MMA (1)
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(ptempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_rank();
  const int leader = rank & ~1;                    // the pair's MMA-issuing CTA
  const bool is_leader = rank == leader;
  const uint16_t pair_mask = (uint16_t)(3u << leader);
  const int64_t ntiles = (n + TM - 1) / TM;
  const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  auto tile_of = [&](int64_t i) { return (cid + i * ncl) * CS + rank; };
  const int64_t iters = ntiles > cid * CS ? (ntiles - cid * CS + ncl * CS - 1) / (ncl * CS) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P256_XR; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 4);
    }
    for (int s = 0; s < P256_OP; ++s) {
      mbar_init(&ofull[s], 4);
      mbar_init(&oempty[s], 1);
    }
    for (int s = 0; s < P256_FR; ++s) {
      mbar_init(&ffull[s], 1);
      mbar_init(&fempty[s], CS / 2);
    }
    for (int s = 0; s < P256_PR; ++s) mbar_init(&pready[s], 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
      mbar_init(&ptempty[a], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;
  if (warp == 0) {
    // ===== X producer: raw fp32 K slices of this CTA's tiles
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t i = 0; i < iters; ++i) {
        const int64_t t = tile_of(i) < ntiles ? tile_of(i) : ntiles - 1;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % P256_XR;
          if (it >= P256_XR) mbar_wait(&xempty[s], ((it / P256_XR) - 1) & 1);
          mbar_expect_tx(&xfull[s], CHUNK_BYTES);
          tma_load_2d(sXR + (size_t)s * CHUNK_BYTES, &xmap, kb * B256_KC, (int)(t * TM), &xfull[s]);
        }
      }
    }
  } else if (warp == 10) {
    // ===== F producer: rows [64 rank, +64) of every F^T slice, to the two CTAs
    // that hold that half (pair rank = rank / 2: cluster ranks rank/2 and rank/2 + 2)
    if (lane == 0) {
      const uint16_t fmask = (uint16_t)(5u << (rank >> 1));
      uint32_t it = 0;
      for (int64_t i = 0; i < iters; ++i)
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % P256_FR;
          if (it >= P256_FR) mbar_wait(&fempty[s], ((it / P256_FR) - 1) & 1);
          // this CTA's half of the slice: 128 rows x 64 B, hi and lo
          mbar_expect_tx(&ffull[s], 2 * P256_FH);
          unsigned char* fb = sF + (size_t)s * 2 * P256_FH;
          if (CS == 4) {
            // two source CTAs per half: this one brings rows [64 rank, +64)
            unsigned char* fh = fb + (rank & 1) * 64 * 64;
            tma_load_2d_mc(fh, &fhmap, kb * B256_KC, rank * 64, &ffull[s], fmask);
            tma_load_2d_mc(fh + P256_FH, &flmap, kb * B256_KC, rank * 64, &ffull[s], fmask);
          } else {
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              tma_load_2d(fb + h2 * 64 * 64, &fhmap, kb * B256_KC, rank * 128 + h2 * 64, &ffull[s]);
              tma_load_2d(fb + P256_FH + h2 * 64 * 64, &flmap, kb * B256_KC, rank * 128 + h2 * 64, &ffull[s]);
            }
          }
        }
    }
  } else if (warp == 1) {
    if (lane == 0 && is_leader) {
      // ===== MMA issuer of the pair: M = 256 (128 rows per CTA), N = 256 (128 F rows per CTA)
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(D >> 3) << 17) |
                                 ((uint32_t)((2 * TM) >> 4) << 24);
      uint32_t it = 0, tl = 0;
      const uint32_t obase = smem_u32(sOP), fbase = smem_u32(sF);
      for (int64_t i = 0; i < iters; ++i, ++tl) {
        const int a = tl & 1;
        if (tl >= 2) {
          mbar_wait(&tempty[a], ((tl >> 1) - 1) & 1);
          mbar_wait(&ptempty[a], ((tl >> 1) - 1) & 1);
        }
        tc_fence_after();
        const uint32_t dtm = tmem + (uint32_t)(a * D);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int so = it % P256_OP, sf = it % P256_FR;
          mbar_wait(&ffull[sf], (it / P256_FR) & 1);
          mbar_wait(&ofull[so], (it / P256_OP) & 1);
          mbar_wait(&pready[it % P256_PR], (it / P256_PR) & 1);
          tc_fence_after();
          const uint32_t xh = obase + (uint32_t)so * 2 * 8192, xl = xh + 8192;
          const uint32_t fh = fbase + (uint32_t)sf * 2 * P256_FH, fl = fh + P256_FH;
#pragma unroll
          for (int ks = 0; ks < B256_KC / 16; ++ks) {  // 16 bf16 (32 B) per MMA
            const uint32_t ko = ks * 32;
            const uint32_t acc0 = (kb | ks) ? 1u : 0u;
            mma_bf16_2cta(dtm, umma_desc_sw64(xh + ko), umma_desc_sw64(fh + ko), idesc, acc0);
            mma_bf16_2cta(dtm, umma_desc_sw64(xh + ko), umma_desc_sw64(fl + ko), idesc, 1u);
            mma_bf16_2cta(dtm, umma_desc_sw64(xl + ko), umma_desc_sw64(fh + ko), idesc, 1u);
          }
          mma_commit_mc2(&oempty[so], pair_mask);
          mma_commit_mc2(&fempty[sf], (uint16_t)((1u << CS) - 1));
        }
        mma_commit_mc2(&tfull[a], pair_mask);
      }
    } else if (lane == 0) {
      // ===== the peer's forwarder: one cluster-scope arrival per slice ("my
      // operands and my F half are in place") and per drained accumulator, so
      // that the split and epilogue warps signal locally (a release at cluster
      // scope from every warp cost 28 % of the kernel's issue slots in fences)
      uint32_t it = 0, tl = 0;
      for (int64_t i = 0; i < iters; ++i, ++tl) {
        const int a = tl & 1;
        if (tl >= 2) {
          mbar_wait(&tempty[a], ((tl >> 1) - 1) & 1);
          mbar_arrive_cta(&ptempty[a], (uint32_t)leader);
        }
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int so = it % P256_OP, sf = it % P256_FR;
          mbar_wait(&ffull[sf], (it / P256_FR) & 1);
          mbar_wait(&ofull[so], (it / P256_OP) & 1);
          mbar_arrive_cta(&pready[it % P256_PR], (uint32_t)leader);
        }
      }
    }
  } else if (warp < 6) {
    // ===== split (as in the single-CTA kernel); "operands ready" goes to the leader
    const int r = threadIdx.x - 64;
    const uint32_t xbase = smem_u32(sXR), obase = smem_u32(sOP);
    uint32_t it = 0;
    for (int64_t i = 0; i < iters; ++i)
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const int sx = it % P256_XR, so = it % P256_OP;
        mbar_wait(&xfull[sx], (it / P256_XR) & 1);
        const uint32_t st = xbase + (uint32_t)sx * CHUNK_BYTES;
        float4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = lds128(st + r * 128 + ((c ^ (r & 7)) << 4));
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[sx]);  // raw slot free: values are in registers
        if (it >= P256_OP) mbar_wait(&oempty[so], ((it / P256_OP) - 1) & 1);
        const uint32_t ob = obase + (uint32_t)so * 2 * 8192;
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // bf16 chunk c = fp32 columns 8c .. 8c+7
          const float4 p = v[2 * c], q = v[2 * c + 1];
          uint4 h, l;
          h.x = pack_bf16(p.x, p.y);
          h.y = pack_bf16(p.z, p.w);
          h.z = pack_bf16(q.x, q.y);
          h.w = pack_bf16(q.z, q.w);
          l.x = pack_bf16(p.x - __uint_as_float(h.x << 16), p.y - __uint_as_float(h.x & 0xFFFF0000u));
          l.y = pack_bf16(p.z - __uint_as_float(h.y << 16), p.w - __uint_as_float(h.y & 0xFFFF0000u));
          l.z = pack_bf16(q.x - __uint_as_float(h.z << 16), q.y - __uint_as_float(h.z & 0xFFFF0000u));
          l.w = pack_bf16(q.z - __uint_as_float(h.w << 16), q.w - __uint_as_float(h.w & 0xFFFF0000u));
          const uint32_t off = r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
          sts128(ob + off, h);
          sts128(ob + 8192 + off, l);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ofull[so]);
      }
  } else {
    // ===== epilogue: TMEM -> registers -> swizzled smem -> TMA store (this CTA's 128 rows)
    const int q = warp & 3;
    unsigned char* stg = sO + (size_t)(warp - 6) * 2 * OSTAGE;
    uint32_t tl = 0, sb = 0;
    for (int64_t i = 0; i < iters; ++i, ++tl) {
      const int64_t t = tile_of(i);
      const int a = tl & 1;
      mbar_wait(&tfull[a], (tl >> 1) & 1);
      tc_fence_after();
      const int64_t row0 = t * TM + q * 32;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32, sb ^= 1) {
        uint32_t rr[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * D + c0), rr);
        unsigned char* buf = stg + sb * OSTAGE;
        if (lane == 0) tma_store_wait_read1();
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(buf + sw128(lane, 4 * v)) =
              make_float4(__uint_as_float(rr[4 * v]), __uint_as_float(rr[4 * v + 1]),
                          __uint_as_float(rr[4 * v + 2]), __uint_as_float(rr[4 * v + 3]));
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && row0 < n) tma_store_2d(&zmap, c0, (int)row0, buf);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    if (lane == 0) tma_store_wait_all();
  }
  tc_fence_before();
  // no CTA may leave while a peer can still multicast into it or arrive on its barriers
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int CS>
cudaError_t launch_bf16_256(const CUtensorMap& map, const CUtensorMap& zm, const CUtensorMap& fh,
                            const CUtensorMap& fl, int64_t n, int64_t ntiles, cudaStream_t s, int nsm) {
  const size_t smem = B256_SMEM;
  static int grid = 0;
  if (!grid) {
    cudaError_t e = cudaFuncSetAttribute(materialize_bf16_256<CS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    grid = nsm / CS * CS;
    if (CS > 1) {  // clusters live inside a GPC: use as many as fit at once
      cudaLaunchConfig_t q = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.gridDim = dim3(grid);
      q.blockDim = dim3(B256_THREADS);
      q.dynamicSmemBytes = smem;
      q.attrs = at;
      q.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, materialize_bf16_256<CS>, &q) == cudaSuccess && ncl > 0 &&
          ncl * CS < grid)
        grid = ncl * CS;
    }
  }
  int g = grid;
  const int64_t groups = (ntiles + CS - 1) / CS;
  if (groups * CS < g) g = (int)(groups * CS);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(B256_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, materialize_bf16_256<CS>, map, zm, fh, fl, n);
}

template <int CS>
cudaError_t launch_bf16_256_pair(const CUtensorMap& map, const CUtensorMap& zm, const CUtensorMap& fh,
                                 const CUtensorMap& fl, int64_t n, int64_t ntiles, cudaStream_t s, int nsm) {
  const size_t smem = P256_SMEM;
  static int grid = 0;
  if (!grid) {
    cudaError_t e = cudaFuncSetAttribute(materialize_bf16_256_pair<CS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    grid = nsm / CS * CS;
    cudaLaunchConfig_t q = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    q.gridDim = dim3(grid);
    q.blockDim = dim3(B256_THREADS);
    q.dynamicSmemBytes = smem;
    q.attrs = at;
    q.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, materialize_bf16_256_pair<CS>, &q) == cudaSuccess && ncl > 0 &&
        ncl * CS < grid)
      grid = ncl * CS;
  }
  int g = grid;
  const int64_t groups = (ntiles + CS - 1) / CS;
  if (groups * CS < g) g = (int)(groups * CS);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(B256_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, materialize_bf16_256_pair<CS>, map, zm, fh, fl, n);
}

template <int D>
size_t tc_smem() {
  return 1024 + 2 * (D / KC) * (D * KC * 4) + stages_for<D>() * 2 * CHUNK_BYTES + 8 * OSTAGE + 256;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int D>
cudaError_t launch_tc(const float* X, int64_t n, int ldx, const float* Fhi, const float* Flo,
                      float* Z, int ldz, cudaStream_t s, int nsm) {
  auto encode = get_encode();
  if (!encode) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
  cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)TM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  CUtensorMap zm;
  cuuint64_t zdims[2] = {(cuuint64_t)D, (cuuint64_t)n};
  cuuint64_t zstr[1] = {(cuuint64_t)ldz * 4};
  cuuint32_t zbox[2] = {(cuuint32_t)KC, 32u};
  r = encode(&zm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Z, zdims, zstr, zbox, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  const int64_t ntiles = (n + TM - 1) / TM;
  const int grid = (int)(ntiles < nsm ? ntiles : nsm);
  if (D == 256) {
    // Fhi / Flo hold bf16 [256][256] (FT layout) for this path
    CUtensorMap fh, fl;
    cuuint64_t fdims[2] = {256, 256};
    cuuint64_t fstr[1] = {256 * 2};
    cuuint32_t fbox[2] = {(cuuint32_t)B256_KC, (cuuint32_t)(256 / B256_CS)};
    r = encode(&fh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<float*>(Fhi), fdims, fstr, fbox,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    r = encode(&fl, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<float*>(Flo), fdims, fstr, fbox,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    // dev switch while the pair kernel is being validated: DAMF_MAT256_PAIR=1
    static const int pair = [] { const char* e = getenv("DAMF_MAT256_PAIR"); return e ? atoi(e) : 4; }();
    static_assert(B256_CS == 4, "the pair kernel shares the 64-row F boxes of the 4-CTA clusters");
    if (pair == 4) return launch_bf16_256_pair<4>(map, zm, fh, fl, n, ntiles, s, nsm);
    if (pair == 2) return launch_bf16_256_pair<2>(map, zm, fh, fl, n, ntiles, s, nsm);
    return launch_bf16_256<B256_CS>(map, zm, fh, fl, n, ntiles, s, nsm);
  }
  if (D == 128) {
    const size_t smem = 1024 + TS_STAGES * 2 * CHUNK_BYTES + 8 * OSTAGE + 256;
    static bool cfg128 = false;
    if (!cfg128) {
      cudaError_t e = cudaFuncSetAttribute(materialize_tc128_ts,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      cfg128 = true;
    }
    materialize_tc128_ts<<<grid, THREADS, smem, s>>>(map, zm, Fhi, Flo, n);
    return cudaGetLastError();
  }
  const size_t smem = tc_smem<D>();
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(materialize_tc_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  materialize_tc_kernel<D><<<grid, THREADS, smem, s>>>(map, zm, Fhi, Flo, n);
  return cudaGetLastError();
}

}  // namespace

bool materialize_tc_supported(int k, int ldx, int ldz, const void* X, const void* Z) {
  return (k == 32 || k == 64 || k == 128 || k == 256) && (ldx % 4) == 0 && (ldz % 4) == 0 &&
         ((uintptr_t)X % 16) == 0 && ((uintptr_t)Z % 16) == 0;
}

// Fhi/Flo: device fp32 arrays of k*k, row j = output column j (FT layout).
cudaError_t launch_materialize_tc(const float* X, int64_t n, int k, int ldx, const float* Fhi,
                                  const float* Flo, float* Z, int ldz, cudaStream_t s, int nsm) {
  if (n <= 0) return cudaSuccess;
  switch (k) {
    case 32: return launch_tc<32>(X, n, ldx, Fhi, Flo, Z, ldz, s, nsm);
    case 64: return launch_tc<64>(X, n, ldx, Fhi, Flo, Z, ldz, s, nsm);
    case 128: return launch_tc<128>(X, n, ldx, Fhi, Flo, Z, ldz, s, nsm);
    case 256: return launch_tc<256>(X, n, ldx, Fhi, Flo, Z, ldz, s, nsm);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dgpu
