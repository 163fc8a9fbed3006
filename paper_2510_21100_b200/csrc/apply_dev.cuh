// apply_dev.cuh -- device helpers of kernel (d): the exact integer colour reconstruction and
// the TMA bulk-copy / mbarrier PTX wrappers, used by k_apply (k_apply.cu).
//
// P:308 ("we utilize the histogram matching to estimate the enhanced image") and P:59
// (S is the HSV value channel): V = max(R,G,B), V' = LUT[V]; replacing V in hexcone HSV
// scales every channel by V'/V (reading R17), rounded half up:
//     out_c = floor((2 c V' + V) / (2 V)),  V = 0 -> (V', V', V').
// Integer form (the scalar kernel): out_c = umulhi(c * e + V, M[V]) + (e >> 16) with
//     V >= 1: e = 2 LUT[V],  M = floor(2^32 / (2V)) + 1   (exact for every numerator <= 130305)
//     V == 0: e = LUT[0] << 16 (then c = 0, the numerator is 0 and the addend gives LUT[0]).
// fp32 form (the streaming kernel): out_c = rn(c alpha + beta), below.
//
// B200 design: every warp runs its own TMA bulk-copy pipeline over 1024-pixel chunks
// (3,072 B): cp.async.bulk global->smem completes on a per-stage mbarrier, the 32 lanes
// transform the chunk in place as two 512-px sub-blocks (lane l owns 16 px of each: three
// conflict-free 16-B LDS/STS at a 48-B lane stride), and cp.async.bulk smem->global writes
// whole lines back -- no partial-sector stores.  Per pixel one 8-B LDS fetches (alpha, beta) from
// a per-warp table rebuilt when the warp's chunk changes image, so warps never synchronise with
// each other.  Chunks never straddle images; images whose pixel count is not a multiple of 16
// (or unaligned buffers) take the scalar kernel.
#pragma once
#include "hr_common.cuh"

namespace hr {
namespace {

constexpr int kWarps = kApplyThreads / 32;
constexpr int kSubPx = 512;                 // px per sub-block: lane l owns [16 l, 16 l + 16)
constexpr int kSubBytes = kSubPx * 3;       // 1536
constexpr int kChunkPx = 2 * kSubPx;        // px per bulk copy
constexpr int kChunkBytes = kChunkPx * 3;   // 3072
constexpr int kStages = 4;
constexpr int kAhead = kStages - 2;  // chunks prefetched ahead of the one being computed

__device__ __forceinline__ uint32_t bx(uint32_t w, int k) { return __byte_perm(w, 0u, 0x4440u | (uint32_t)k); }

__host__ __device__ constexpr uint32_t magic_of(int v) {
  return v == 0 ? 0u : (uint32_t)(0x100000000ull / (uint64_t)(2 * v)) + 1u;
}
__host__ __device__ constexpr uint32_t ab_of(int v, uint32_t L) { return v == 0 ? (L << 16) : (2u * L); }

// one pixel channel, integer form (the scalar fallback kernel):
// floor((2 c V' + V) / 2V) = umulhi(c*e + V, M) + F
__device__ __forceinline__ uint32_t chan(uint32_t c, uint32_t e, uint32_t v, uint32_t M, uint32_t F) {
  return __umulhi(c * e + v, M) + F;
}

// The streaming kernel evaluates the same quotient in fp32 (IMAD.HI issues at a quarter of the
// FFMA rate on this part: 4.1 vs 1.1-2 cycles per warp instruction per scheduler,
// tools/imad_probe.cu): per level V the table holds alpha = fl(V'/V) and beta = fl(1 / 4V), and
// out_c = rn(c alpha + beta) = rn((2cV' + V + 1/2) / 2V - 1/2).  Exact: (2cV' + V + 1/2) / 2V lies at least 1/(4V) >=
// 9.8e-4 from every integer, the fp32 error of c alpha + beta is <= 5e-5, so rounding to nearest
// of the value minus 1/2 is the floor (checked exhaustively over every V, c <= V, V' on the
// host and against the oracle on the GPU).  Bytes enter as "magic" floats 2^23 + c (one PRMT
// builds the bit pattern), leave as the low mantissa byte of (c alpha + beta) + 1.5 * 2^23.
// (beta = (V + 1/2) / 2V - 1/2 = 1 / 4V.)  V == 0: alpha = 0, beta = V'.
constexpr uint32_t kMagicBits = 0x4B000000u;  // 2^23 as float bits
__device__ __forceinline__ uint32_t mg(uint32_t w, int k) { return __byte_perm(w, kMagicBits, 0x7540u | (uint32_t)k); }
__device__ __forceinline__ uint2 tab_entry(int v, uint32_t L) {
  if (v == 0) return make_uint2(0u, __float_as_uint((float)L));
  // the correctly rounded fp32 quotients V'/V and 1/(4V) (IEEE division: the host check's values;
  // no constant table: after an L2 flush its loads would be DRAM misses on a single image's
  // critical path); the divisions see normal operands only (a zero numerator takes a slow path)
  const float fv = (float)v;
  const float a = __fdiv_rn((float)(L ? L : 1u), fv);
  return make_uint2(L ? __float_as_uint(a) : 0u, __float_as_uint(__fdiv_rn(0.25f, fv)));
}
// out byte (in the low byte of the returned bits) of channel magic float cm
__device__ __forceinline__ uint32_t chanf(uint32_t cm, float alpha, float beta) {
  const float c = __uint_as_float(cm) - 8388608.0f;
  return __float_as_uint(fmaf(c, alpha, beta) + 12582912.0f);
}

// 4 pixels in 3 words -> 3 words.  tab_s: shared-window address of the per-warp (alpha, beta)
// table minus 8 * 0x4B000000 (mod 2^32), so the entry of a magic-float level v is at v * 8 + tab_s.
__device__ __forceinline__ void apply4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t tab_s, uint32_t& o0,
                                       uint32_t& o1, uint32_t& o2) {
  const uint32_t r0 = mg(w0, 0), g0 = mg(w0, 1), b0 = mg(w0, 2);
  const uint32_t r1 = mg(w0, 3), g1 = mg(w1, 0), b1 = mg(w1, 1);
  const uint32_t r2 = mg(w1, 2), g2 = mg(w1, 3), b2 = mg(w2, 0);
  const uint32_t r3 = mg(w2, 1), g3 = mg(w2, 2), b3 = mg(w2, 3);
  // the magic floats share their upper 24 bits: the integer maximum is the maximum byte
  const uint32_t v0 = __vimax3_u32(r0, g0, b0), v1 = __vimax3_u32(r1, g1, b1);
  const uint32_t v2 = __vimax3_u32(r2, g2, b2), v3 = __vimax3_u32(r3, g3, b3);
  float a0, e0, a1, e1, a2, e2, a3, e3;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a0), "=f"(e0) : "r"(v0 * 8u + tab_s));
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a1), "=f"(e1) : "r"(v1 * 8u + tab_s));
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a2), "=f"(e2) : "r"(v2 * 8u + tab_s));
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a3), "=f"(e3) : "r"(v3 * 8u + tab_s));
  const uint32_t R0 = chanf(r0, a0, e0), G0 = chanf(g0, a0, e0), Q0 = chanf(b0, a0, e0);
  const uint32_t R1 = chanf(r1, a1, e1), G1 = chanf(g1, a1, e1), Q1 = chanf(b1, a1, e1);
  const uint32_t R2 = chanf(r2, a2, e2), G2 = chanf(g2, a2, e2), Q2 = chanf(b2, a2, e2);
  const uint32_t R3 = chanf(r3, a3, e3), G3 = chanf(g3, a3, e3), Q3 = chanf(b3, a3, e3);
  o0 = __byte_perm(__byte_perm(R0, G0, 0x3340u), __byte_perm(Q0, R1, 0x3340u), 0x5410u);
  o1 = __byte_perm(__byte_perm(G1, Q1, 0x3340u), __byte_perm(R2, G2, 0x3340u), 0x5410u);
  o2 = __byte_perm(__byte_perm(Q2, R3, 0x3340u), __byte_perm(G3, Q3, 0x3340u), 0x5410u);
}

// per-warp (alpha, beta) table of image b's LUT (lut read through L2: it may have been written by
// another CTA of the same launch); the caller __syncwarp()s around it
__device__ __forceinline__ void build_tab(uint2* tab, const uint8_t* __restrict__ lut_b, int lane) {
  uint32_t L[kLevels / 32];
#pragma unroll
  for (int i = 0; i < kLevels / 32; ++i) L[i] = __ldcg(lut_b + lane + 32 * i);  // the loads in flight together
#pragma unroll 2
  for (int i = 0; i < kLevels / 32; ++i) tab[lane + 32 * i] = tab_entry(lane + 32 * i, L[i]);
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
  uint8_t stage[kWarps][kStages][kChunkBytes];  // 96 KB
  uint2 tab[kWarps][kLevels];                   // 16 KB: per-warp (alpha, beta) as float bits
  uint64_t bar[kWarps][kStages];
};

// One staged chunk (<= 1024 px at p, `bytes` valid, a multiple of 48) transformed in place:
// sub-block h in [0, 2), lane l owns pixels [512 h + 16 l, 512 h + 16 l + 16).
__device__ __forceinline__ void apply_chunk_smem(uint8_t* p, uint32_t bytes, const uint2* __restrict__ tab, int lane) {
  const uint32_t tab_s = smem_u32(tab) - 0x58000000u;  // - 8 * 0x4B000000 (mod 2^32)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t o = (uint32_t)h * kSubBytes + (uint32_t)lane * 48u;
    if (o < bytes) {
      uint4* q = reinterpret_cast<uint4*>(p + o);
      const uint4 a = q[0], c = q[1], d = q[2];
      uint4 x, y, z;
      apply4(a.x, a.y, a.z, tab_s, x.x, x.y, x.z);
      apply4(a.w, c.x, c.y, tab_s, x.w, y.x, y.y);
      apply4(c.z, c.w, d.x, tab_s, y.z, y.w, z.x);
      apply4(d.y, d.z, d.w, tab_s, z.y, z.z, z.w);
      q[0] = x;
      q[1] = y;
      q[2] = z;
    }
  }
}

}  // namespace
}  // namespace hr
