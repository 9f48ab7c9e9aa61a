// gss_device.cuh — sm_100a device primitives for the survival-scan kernels:
// mbarrier / TMA (cp.async.bulk.tensor) wrappers, gpu-scope acquire/release
// flag access for the decoupled look-back, and the segmented lane algebra.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace gss {

// ---------------------------------------------------------------------------
// geometry (fixed at pack time: tile-blocked column pointers depend on it)
// ---------------------------------------------------------------------------
constexpr int kIpt = 8;                     // rows per lane per pass
constexpr int kTileRows = 2048;             // rows per tile (8 passes x 32 lanes x 8 rows)
constexpr int kPasses = kTileRows / (32 * kIpt);
constexpr int kNnzCap = 256;                // per-list smem capacity (ints) of a column's
                                            // in-tile nonzero list

// per-row code word (uint32): built per engine from times/status/mask/strata
constexpr uint32_t kCodeCount = 0x0FFFFFFFu;  // events in the tied block, at its last row
constexpr uint32_t kCodeCompeting = 1u << 28; // status==2 and visible (Fine-Gray u row)
constexpr uint32_t kCodeMasked = 1u << 29;    // row not visible to this engine (or padding)
constexpr uint32_t kCodeEvent = 1u << 30;     // status==1 and visible (for sum delta*eta)
constexpr uint32_t kCodeSeg = 1u << 31;       // first row of a stratum

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// One non-blocking probe of a phase (for lane-divergent waits: the retry loop
// stays visible to the compiler, so divergent lanes keep making progress).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// TMA 2D tile load (global -> shared), completion counted on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 1D bulk copy (global -> shared); bytes % 16 == 0, both addresses 16B aligned.
__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// gpu-scope release store / acquire load of a 64-bit status word
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// coherent (L1-bypassing) payload load
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Swizzled byte offset inside a TMA box whose rows are W bytes wide and were
// loaded with CU_TENSOR_MAP_SWIZZLE_{W}B (W in {32, 64, 128}): the 16-byte
// chunk index (bits [4, 4+log2(W/16))) is XORed with bits [7, ...).
template <int W>
__device__ __forceinline__ uint32_t swz(uint32_t off) {
  return off ^ (((off >> 7) & (W / 16 - 1)) << 4);
}

// ---------------------------------------------------------------------------
// Segmented lane algebra.  A value (f, v[L]) is the sum of a run of rows;
// f = "the run contains the first row of a stratum".  Combining an earlier
// run x with a later run y:  (x.f | y.f,  y.f ? y.v : x.v + y.v).
// Associative; (0, 0...) is the identity, and adding +0.0 is exact, so
// inactive slots never perturb a sum.
// ---------------------------------------------------------------------------
template <int L>
struct Seg {
  uint32_t f;
  double v[L];
  __device__ __forceinline__ static Seg zero() {
    Seg s;
    s.f = 0;
#pragma unroll
    for (int i = 0; i < L; ++i) s.v[i] = 0.0;
    return s;
  }
};

template <int L>
__device__ __forceinline__ Seg<L> seg_combine(const Seg<L>& x, const Seg<L>& y) {
  Seg<L> r;
  r.f = x.f | y.f;
#pragma unroll
  for (int i = 0; i < L; ++i) r.v[i] = y.f ? y.v[i] : __dadd_rn(x.v[i], y.v[i]);
  return r;
}

template <int L>
__device__ __forceinline__ Seg<L> shfl_up_seg(const Seg<L>& s, int delta) {
  Seg<L> r;
  r.f = __shfl_up_sync(0xffffffffu, s.f, delta);
#pragma unroll
  for (int i = 0; i < L; ++i) r.v[i] = __shfl_up_sync(0xffffffffu, s.v[i], delta);
  return r;
}

template <int L>
__device__ __forceinline__ Seg<L> shfl_down_seg(const Seg<L>& s, int delta) {
  Seg<L> r;
  r.f = __shfl_down_sync(0xffffffffu, s.f, delta);
#pragma unroll
  for (int i = 0; i < L; ++i) r.v[i] = __shfl_down_sync(0xffffffffu, s.v[i], delta);
  return r;
}

// Inclusive warp scan (fixed shuffle tree => deterministic).
template <int L>
__device__ __forceinline__ Seg<L> warp_inclusive_scan(Seg<L> s, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Seg<L> o = shfl_up_seg(s, d);
    if (lane >= d) s = seg_combine(o, s);
  }
  return s;
}

// Ordered warp reduction: lane 0 gets lane0 ⊕ lane1 ⊕ ... ⊕ lane31 (tree order).
template <int L>
__device__ __forceinline__ Seg<L> warp_ordered_reduce(Seg<L> s) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Seg<L> o = shfl_down_seg(s, d);
    s = seg_combine(s, o);  // lanes beyond 31-d read their own value; unused
  }
  return s;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

}  // namespace gss
