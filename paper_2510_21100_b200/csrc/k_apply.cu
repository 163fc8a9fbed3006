// k_apply.cu -- kernel (d): streaming LUT application + colour reconstruction.
//
// P:308 ("we utilize the histogram matching to estimate the enhanced image") and P:59
// (S is the HSV value channel): V = max(R,G,B), V' = LUT[V]; replacing V in hexcone HSV
// scales every channel by V'/V (reading R17), rounded half up:
//     out_c = floor((2 c V' + V) / (2 V)),  V = 0 -> (V', V', V').
// Exact integer form: out_c = umulhi(c * e + V, M[V]) + (e >> 16) with the per-level entry
//     V >= 1: e = 2 LUT[V],  M = floor(2^32 / (2V)) + 1   (exact for every numerator <= 130305)
//     V == 0: e = LUT[0] << 16 (then c = 0, the numerator is 0 and the addend gives LUT[0]),
// i.e. one IMAD and one IMAD.HI (with addend) per channel.
//
// B200 design: every warp runs its own TMA bulk-copy pipeline over 512-pixel chunks
// (1,536 B): cp.async.bulk global->smem completes on a per-stage mbarrier, the 32 lanes
// transform their 16 pixels in place (three conflict-free 16-B LDS/STS at a 48-B lane
// stride), and cp.async.bulk smem->global writes whole lines back -- no partial-sector
// stores (the v1 per-thread 48-B STG pattern sent 1.4x the bytes to L2).  M lives in a
// lane-private table (word 32v + lane: conflict-free), (A | Bv << 16) in a per-warp table
// rebuilt when the warp's chunk changes image, so warps never synchronise with each other.
// Chunks never straddle images; images whose pixel count is not a multiple of 16 (or
// unaligned buffers) take the scalar fallback kernel.
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int kWarps = kApplyThreads / 32;
constexpr int kChunkPx = 512;
constexpr int kChunkBytes = kChunkPx * 3;  // 1536
constexpr int kStages = 5;
constexpr int kAhead = kStages - 2;  // chunks prefetched ahead of the one being computed

__device__ __forceinline__ uint32_t bx(uint32_t w, int k) { return __byte_perm(w, 0u, 0x4440u | (uint32_t)k); }

__device__ __forceinline__ uint32_t magic_of(int v) {
  return v == 0 ? 0u : (uint32_t)(0x100000000ull / (uint64_t)(2 * v)) + 1u;
}
__device__ __forceinline__ uint32_t ab_of(int v, uint32_t L) { return v == 0 ? (L << 16) : (2u * L); }

// one pixel channel: floor((2 c V' + V) / 2V) = umulhi(c*e + V, M) + F
__device__ __forceinline__ uint32_t chan(uint32_t c, uint32_t e, uint32_t v, uint32_t M, uint32_t F) {
  return __umulhi(c * e + v, M) + F;
}

// 4 pixels in 3 words -> 3 words.  ab: per-warp table, mt: lane-private magic table.
__device__ __forceinline__ void apply4(uint32_t w0, uint32_t w1, uint32_t w2, const uint32_t* __restrict__ ab,
                                       const uint32_t* __restrict__ mt, int lane, uint32_t& o0, uint32_t& o1,
                                       uint32_t& o2) {
  const uint32_t r0 = bx(w0, 0), g0 = bx(w0, 1), b0 = bx(w0, 2);
  const uint32_t r1 = bx(w0, 3), g1 = bx(w1, 0), b1 = bx(w1, 1);
  const uint32_t r2 = bx(w1, 2), g2 = bx(w1, 3), b2 = bx(w2, 0);
  const uint32_t r3 = bx(w2, 1), g3 = bx(w2, 2), b3 = bx(w2, 3);
  const uint32_t v0 = __vimax3_u32(r0, g0, b0), v1 = __vimax3_u32(r1, g1, b1);
  const uint32_t v2 = __vimax3_u32(r2, g2, b2), v3 = __vimax3_u32(r3, g3, b3);
  const uint32_t e0 = ab[v0], e1 = ab[v1], e2 = ab[v2], e3 = ab[v3];
  const uint32_t m0 = mt[(v0 << 5) | lane], m1 = mt[(v1 << 5) | lane];
  const uint32_t m2 = mt[(v2 << 5) | lane], m3 = mt[(v3 << 5) | lane];
  const uint32_t F0 = e0 >> 16, F1 = e1 >> 16, F2 = e2 >> 16, F3 = e3 >> 16;
  const uint32_t R0 = chan(r0, e0, v0, m0, F0), G0 = chan(g0, e0, v0, m0, F0), Q0 = chan(b0, e0, v0, m0, F0);
  const uint32_t R1 = chan(r1, e1, v1, m1, F1), G1 = chan(g1, e1, v1, m1, F1), Q1 = chan(b1, e1, v1, m1, F1);
  const uint32_t R2 = chan(r2, e2, v2, m2, F2), G2 = chan(g2, e2, v2, m2, F2), Q2 = chan(b2, e2, v2, m2, F2);
  const uint32_t R3 = chan(r3, e3, v3, m3, F3), G3 = chan(g3, e3, v3, m3, F3), Q3 = chan(b3, e3, v3, m3, F3);
  o0 = __byte_perm(__byte_perm(R0, G0, 0x3340u), __byte_perm(Q0, R1, 0x3340u), 0x5410u);
  o1 = __byte_perm(__byte_perm(G1, Q1, 0x3340u), __byte_perm(R2, G2, 0x3340u), 0x5410u);
  o2 = __byte_perm(__byte_perm(Q2, R3, 0x3340u), __byte_perm(G3, Q3, 0x3340u), 0x5410u);
}

// ---- PTX wrappers: mbarrier + bulk async copies (sm_90+, used on sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

struct __align__(128) ApplySmem {
  uint8_t stage[kWarps][kStages][kChunkBytes];  // 60 KB
  uint32_t mt[kLevels * 32];                    // 32 KB lane-private magic
  uint32_t ab[kWarps][kLevels];                 // 8 KB per-warp (A | Bv << 16)
  uint64_t bar[kWarps][kStages];
};

__global__ void __launch_bounds__(kApplyThreads, 2)
k_apply_tma(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t B, int64_t HW,
            uint8_t* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  ApplySmem& s = *reinterpret_cast<ApplySmem*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < kLevels * 32; i += kApplyThreads) s.mt[i] = magic_of(i >> 5);
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&s.bar[w][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t cpi = (uint32_t)((HW + kChunkPx - 1) / kChunkPx);  // chunks per image
  const int64_t G = B * (int64_t)cpi;                               // < 2^31 (host-checked)
  const uint32_t g0 = (uint32_t)(G * blockIdx.x / gridDim.x), g1 = (uint32_t)(G * (blockIdx.x + 1) / gridDim.x);
  // this warp's chunks: g0 + w, g0 + w + kWarps, ...
  const int mine = (g1 - g0 > (uint32_t)w) ? (int)((g1 - g0 - w + kWarps - 1) / kWarps) : 0;
  const uint64_t pol = policy_evict_first();
  uint32_t* ab = s.ab[w];
  int64_t cur_img = -1;

  // chunk cursor: image b, chunk c within the image; advances by kWarps chunks
  struct Cur {
    uint32_t b, c;
  };
  auto start = [&]() {
    const uint32_t g = g0 + (uint32_t)w;
    return Cur{g / cpi, g % cpi};
  };
  auto advance = [&](Cur& k) {
    k.c += kWarps;
    while (k.c >= cpi) {
      k.c -= cpi;
      ++k.b;
    }
  };
  auto where = [&](const Cur& k, uint64_t& off, uint32_t& bytes) {
    const uint32_t px0 = k.c * kChunkPx;
    const uint32_t npx = min((uint32_t)kChunkPx, (uint32_t)(HW - px0));
    off = ((uint64_t)k.b * (uint64_t)HW + px0) * 3u;
    bytes = npx * 3u;
  };
  Cur ld = start(), cp = ld;  // load cursor (lane 0) and compute cursor
  auto issue = [&](int i) {
    uint64_t off;
    uint32_t bytes;
    where(ld, off, bytes);
    const int st = i % kStages;
    mbar_expect_tx(&s.bar[w][st], bytes);
    bulk_load(s.stage[w][st], in + off, bytes, &s.bar[w][st], pol);
    advance(ld);
  };

  if (lane == 0)
    for (int i = 0; i < min(kAhead, mine); ++i) issue(i);

  int st = 0;
  uint32_t ph = 0;
  for (int i = 0; i < mine; ++i) {
    uint64_t off;
    uint32_t bytes;
    where(cp, off, bytes);
    if ((int64_t)cp.b != cur_img) {  // per-warp LUT table for this image
      __syncwarp();
      for (int v = lane; v < kLevels; v += 32) ab[v] = ab_of(v, lut[(uint64_t)cp.b * kLevels + v]);
      __syncwarp();
      cur_img = cp.b;
    }
    // prefetch chunk i + kAhead into the stage of chunk i - 2, whose bulk store (committed
    // two iterations ago) has finished reading shared memory once all but the latest
    // store group have
    if (lane == 0 && i + kAhead < mine) {
      if (i >= 2) bulk_wait_read<1>();
      issue(i + kAhead);
    }
    mbar_wait(&s.bar[w][st], ph);
    uint8_t* p = s.stage[w][st];
    if ((uint32_t)lane * 48u < bytes) {
      uint4* q = reinterpret_cast<uint4*>(p + lane * 48);
      const uint4 a = q[0], c = q[1], d = q[2];
      uint4 x, y, z;
      apply4(a.x, a.y, a.z, ab, s.mt, lane, x.x, x.y, x.z);
      apply4(a.w, c.x, c.y, ab, s.mt, lane, x.w, y.x, y.y);
      apply4(c.z, c.w, d.x, ab, s.mt, lane, y.z, y.w, z.x);
      apply4(d.y, d.z, d.w, ab, s.mt, lane, z.y, z.z, z.w);
      q[0] = x;
      q[1] = y;
      q[2] = z;
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_store(out + off, p, bytes, pol);
      bulk_commit();
    }
    advance(cp);
    if (++st == kStages) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (lane == 0) bulk_wait<0>();
}

// ---------------------------------------------------------------- scalar fallback
__device__ __forceinline__ void apply_scalar(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t q,
                                             const uint32_t* ab) {
  const uint32_t r = in[3 * q], g = in[3 * q + 1], b = in[3 * q + 2];
  const uint32_t v = __vimax3_u32(r, g, b);
  const uint32_t e = ab[v], M = magic_of((int)v), F = e >> 16;
  out[3 * q] = (uint8_t)chan(r, e, v, M, F);
  out[3 * q + 1] = (uint8_t)chan(g, e, v, M, F);
  out[3 * q + 2] = (uint8_t)chan(b, e, v, M, F);
}

__global__ void __launch_bounds__(kApplyThreads)
k_apply_scalar(const uint8_t* __restrict__ in, const uint8_t* __restrict__ lut, int64_t B, int64_t HW,
               uint8_t* __restrict__ out) {
  __shared__ uint32_t ab[kLevels];
  const int tid = threadIdx.x;
  const int64_t P = B * HW;
  const int64_t q0 = P * blockIdx.x / gridDim.x, q1 = P * (blockIdx.x + 1) / gridDim.x;
  for (int64_t q = q0; q < q1;) {
    const int64_t b = q / HW;
    const int64_t qe = min(q1, (b + 1) * HW);
    __syncthreads();
    ab[tid] = ab_of(tid, lut[b * kLevels + tid]);
    __syncthreads();
    for (int64_t p = q + tid; p < qe; p += kApplyThreads) apply_scalar(in, out, p, ab);
    q = qe;
  }
}

}  // namespace

cudaError_t launch_apply(const uint8_t* in, const uint8_t* lut, int64_t B, int32_t H, int32_t W, uint8_t* out,
                         int grid_ctas, cudaStream_t st) {
  const int64_t HW = (int64_t)H * W;
  const bool tma = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                   (HW % 16 == 0) && B * ((HW + kChunkPx - 1) / kChunkPx) < (1LL << 31);
  if (tma) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_apply_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sizeof(ApplySmem));
      if (e != cudaSuccess) return e;
      attr = true;
    }
    const int64_t chunks = B * ((HW + kChunkPx - 1) / kChunkPx);
    int64_t grid = grid_ctas;
    if (grid > (chunks + kWarps - 1) / kWarps) grid = (chunks + kWarps - 1) / kWarps;
    if (grid < 1) grid = 1;
    k_apply_tma<<<(unsigned)grid, kApplyThreads, sizeof(ApplySmem), st>>>(in, lut, B, HW, out);
  } else {
    int64_t grid = 4LL * grid_ctas;
    const int64_t P = B * HW;
    if (grid > (P + kApplyThreads - 1) / kApplyThreads) grid = (P + kApplyThreads - 1) / kApplyThreads;
    if (grid < 1) grid = 1;
    k_apply_scalar<<<(unsigned)grid, kApplyThreads, 0, st>>>(in, lut, B, HW, out);
  }
  return cudaGetLastError();
}

}  // namespace hr
