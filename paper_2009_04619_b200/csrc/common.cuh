// common.cuh -- device helpers shared by every kernel of the CUDA path:
// mbarrier / TMA PTX wrappers for sm_100a and the per-point arithmetic of one
// time step.  GPU side only; shares nothing with oracle/.
//
// The per-point functions are written with explicit __f*_rn intrinsics so
// that nvcc's FMA contraction cannot differ between inline sites: every
// kernel (naive, interior stream, wall stream, edges/interior split) produces
// bitwise-identical values for the same point, which the 1-GPU == N-slab
// bitwise test relies on.
#pragma once
#include <cstdint>
#include <cuda.h>            // CUtensorMap (type only; no libcuda link)
#include <cuda_runtime.h>

namespace w25 {

constexpr int R = 4;         // stencil radius, PAPER.md L411-414 (R = 4)

// Stencil + PML constants (R8): for fp32 plans fp64-computed and
// rounded once to fp32 on the host; for fp64 plans kept in fp64.  Passed by
// value as a kernel parameter (constant bank).
template <typename T>
struct CoefT {
  T c0;                      // c_xyz
  T cx[R], cy[R], cz[R];     // c_am, m = 1..4
  T i2h[3];                  // 1/(2 h_a)
};
using Coef = CoefT<float>;

// ---------------------------------------------------------------------------
// Per-point arithmetic (SPEC.md L140-157 semantics; fp32 or fp64 with FMA)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// Eq. 3: c_xyz u + sum_m c_am (u(+m) + u(-m)), pair sums
// first (keeps mirror symmetry bitwise), axes x, y, z, m = 1..4.
template <typename T>
struct NbrT { T xm[R], xp[R], ym[R], yp[R], zm[R], zp[R]; };
using Nbr = NbrT<float>;

template <typename T>
__device__ __forceinline__ T lap8(const CoefT<T>& k, T c, const NbrT<T>& n) {
  T L = mul_rn(k.c0, c);
#pragma unroll
  for (int m = 0; m < R; ++m) L = fma_rn(k.cx[m], add_rn(n.xp[m], n.xm[m]), L);
#pragma unroll
  for (int m = 0; m < R; ++m) L = fma_rn(k.cy[m], add_rn(n.yp[m], n.ym[m]), L);
#pragma unroll
  for (int m = 0; m < R; ++m) L = fma_rn(k.cz[m], add_rn(n.zp[m], n.zm[m]), L);
  return L;
}

// inner update, Eq. 2 / SPEC.md L143: (2u - u_prev) + vdt2 L
template <typename T>
__device__ __forceinline__ T upd_inner(T L, T c, T up, T v) {
  return fma_rn(v, L, fma_rn(T(2), c, -up));
}

// one grad-eta . grad-u term: ((eta+ - eta-) / 2h) * ((u+ - u-) / 2h)
template <typename T>
__device__ __forceinline__ T gterm(T ep, T em, T u1p, T u1m, T i2h) {
  return mul_rn(mul_rn(sub_rn(ep, em), i2h), mul_rn(sub_rn(u1p, u1m), i2h));
}

// PML update: ((2u - A u_prev) + vdt2 (L + g)) / B with a true
// IEEE division (a reciprocal multiply drifts past the 1e-5 gate, R9).
// 0 / B (B >= 1) is +-0 exactly; testing for it keeps quiet PML cells (u = 0
// before the wave arrives) off the software slow path of the division.
template <typename T>
__device__ __forceinline__ T upd_pml(T L, T g, T c, T up, T v, T A, T B) {
  const T t = fma_rn(-A, up, mul_rn(T(2), c));
  const T num = fma_rn(v, add_rn(L, g), t);
  return num == T(0) ? num : div_rn(num, B);
}

// ---------------------------------------------------------------------------
// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2: two IEEE fp32 operations
// per instruction, each lane rounded exactly as the scalar instruction -- the
// results are bitwise those of add_rn / mul_rn / fma_rn element by element).
// A pair lives in one 64-bit register pair {lo, hi}.
// ---------------------------------------------------------------------------
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_bcast(float a) { return f2_pack(a, a); }
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
  f2_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// upd_inner on a pair: (2u - up) + v L; 2u is exact, so (u + u) - up rounds
// exactly as fma(2, u, -up)
__device__ __forceinline__ f2_t f2_upd_inner(f2_t L, f2_t c, f2_t up, f2_t v) {
  return f2_fma(v, L, f2_sub(f2_add(c, c), up));
}

// PML division by a TABLE value B with its correctly rounded reciprocal rB =
// RN(1/B) (R9 / SURVEY A20): q0 = RN(n rB), e = RN(n - q0 B) (exact,
// FMA), q = RN(q0 + e rB) -- Markstein's correction, equal to RN(n / B) for
// every n whose result and residual stay normal.  The plan verifies that claim
// EXHAUSTIVELY for its own B values over every fp32 significand at setup
// (k_divcheck; fast = false if any differs), and |n| < 2^-80 (residual could
// be subnormal) takes the IEEE division.  Branch-free on the common path: no
// MUFU, no slow-path call, 3 dependent operations instead of ~10.
template <typename T>
__device__ __forceinline__ T div_table(T n, T B, T rB, bool fast) {
  if (!fast) return n == T(0) ? n : div_rn(n, B);
  const T q0 = mul_rn(n, rB);
  const T q = fma_rn(fma_rn(-q0, B, n), rB, q0);
  if (fabs(n) < T(0x1p-80) && n != T(0)) return div_rn(n, B);
  return n == T(0) ? n : q;        // +-0 / B = +-0 (the formula would give +0 for -0)
}

// div_table on the NV points of a lane, straight-line: all fast quotients
// first (independent chains interleave), then one rarely taken fix-up for
// tiny numerators.  Bitwise div_table per element.  Called by whole warps.
template <typename T, int N>
__device__ __forceinline__ void div_table_row(const T* n, const T* B, const T* rB, bool fast, T* q) {
  if (!fast) {
#pragma unroll
    for (int c = 0; c < N; ++c) q[c] = n[c] == T(0) ? n[c] : div_rn(n[c], B[c]);
    return;
  }
  // a quiet warp (every PML cell the wave has not reached yet: n = +-0 at all
  // its points) skips the quotients: +-0 / B = +-0 (callers are warp-uniform)
  bool z = true;
#pragma unroll
  for (int c = 0; c < N; ++c) z &= n[c] == T(0);
  if (__all_sync(0xffffffffu, z)) {
#pragma unroll
    for (int c = 0; c < N; ++c) q[c] = n[c];
    return;
  }
  bool tiny = false;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    // zeros (every PML cell the wave has not reached) stay on the straight
    // line: +-0 / B = +-0 by a select; only tiny non-zero n branch off
    tiny |= fabs(n[c]) < T(0x1p-80) && n[c] != T(0);
    const T q0 = mul_rn(n[c], rB[c]);
    const T qc = fma_rn(fma_rn(-q0, B[c], n[c]), rB[c], q0);
    q[c] = n[c] == T(0) ? n[c] : qc;
  }
  if (tiny) {
#pragma unroll
    for (int c = 0; c < N; ++c)
      if (fabs(n[c]) < T(0x1p-80) && n[c] != T(0)) q[c] = div_rn(n[c], B[c]);
  }
}

// numerator of the PML update: (2u - A u_prev) + vdt2 (L + g)
template <typename T>
__device__ __forceinline__ T pml_num(T L, T g, T c, T up, T v, T A) {
  return fma_rn(v, add_rn(L, g), fma_rn(-A, up, mul_rn(T(2), c)));
}

// upd_pml with a table B (and its reciprocal): bitwise upd_pml
template <typename T>
__device__ __forceinline__ T upd_pml_t(T L, T g, T c, T up, T v, T A, T B, T rB, bool fast) {
  const T t = fma_rn(-A, up, mul_rn(T(2), c));
  const T num = fma_rn(v, add_rn(L, g), t);
  return div_table(num, B, rB, fast);
}

// 16-byte vector of the precision: 4 floats or 2 doubles per lane
template <typename T> struct VecT;
template <> struct VecT<float> { using V = float4; static constexpr int N = 4; };
template <> struct VecT<double> { using V = double2; static constexpr int N = 2; };

__device__ __forceinline__ float vget(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}
__device__ __forceinline__ double vget(const double2& v, int c) { return c == 0 ? v.x : v.y; }
template <typename T> __device__ __forceinline__ typename VecT<T>::V vmake(const T* a);
template <> __device__ __forceinline__ float4 vmake<float>(const float* a) { return make_float4(a[0], a[1], a[2], a[3]); }
template <> __device__ __forceinline__ double2 vmake<double>(const double* a) { return make_double2(a[0], a[1]); }

// Distance (cells) to the inner box along one axis: 0 inside [w, n-w), 1..w
// in the PML, w+1 outside the domain (eta = 0; clamped so that points of a
// ragged tile beyond the grid index the (w+2)-entry tables safely).
__device__ __forceinline__ int dist1(int i, int n, int w) {
  return min(max(max(w - i, 0), i - (n - w - 1)), w + 1);
}

// ---------------------------------------------------------------------------
// PTX wrappers: shared-memory address, mbarrier, TMA (cp.async.bulk.tensor)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W25_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W25_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 3-D tiled TMA load of one box into shared memory, completion signalled on
// `bar` via complete_tx (bytes).  Out-of-bounds elements are zero-filled --
// this supplies the x/y Dirichlet fringe for free.
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ---- thread-block clusters (DSMEM mbarriers, TMA multicast) ---------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// all threads of all CTAs of the cluster (release / acquire at cluster scope)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of `p`'s offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
  return remote;
}

// arrive on a cluster mbarrier given by its shared::cluster address (default
// .release.cta semantics, as CUTLASS's pipeline consumer_release: a
// cluster-scope release would also drain this warp's outstanding global
// stores before every arrive)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// wait with cluster-scope acquire (the arrivals come from other CTAs' threads)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W25_WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W25_WAITC_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// generic-proxy accesses (any state space, incl. other CTAs' shared memory
// released to us) ordered before our subsequent async-proxy (TMA) operations
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

// TMA load of one box multicast to the CTAs of `cta_mask`: the data lands at
// the same shared-memory offset in each, and each one's mbarrier at `bar`'s
// offset receives the complete_tx bytes.
__device__ __forceinline__ void tma_load_3d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int x,
                                               int y, int z, uint16_t cta_mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6, %7;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "h"(cta_mask),
      "l"(policy)
      : "memory");
}

// L2 prefetch of a 3-D box (no shared memory, no completion tracking): warms
// L2 for a plane the TMA ring will load a few iterations later.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z) : "memory");
}

// Streaming 16-B store (evict-first: u_next is not re-read this step).
__device__ __forceinline__ void st_cs_f4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w) : "memory");
}
__device__ __forceinline__ void st_cs_v(float* p, float4 v) { st_cs_f4(p, v); }
__device__ __forceinline__ void st_cs_v(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <typename T>
__device__ __forceinline__ typename VecT<T>::V ldv(const T* p) {
  return *reinterpret_cast<const typename VecT<T>::V*>(p);
}

__device__ __forceinline__ float f4get(const float4& v, int c) { return vget(v, c); }

}  // namespace w25
