// aux_kernels.cuh -- the non-streaming kernels of the CUDA path: naive
// one-thread-per-point step (the paper's gmem code shape, PAPER.md L429-451;
// ablation / debugging path, bitwise equal to the streaming kernels), source
// injection, medium preparation, finite check.
#pragma once
#include "common.cuh"

namespace w25 {

struct NaiveParams {
  int64_t pitch, plane;
  int nx, ny, nzl, nzg, zoff, w;
  int z0;                      // first local plane of this launch (gridDim.z planes)
  Coef k;                      // fp32 plans
  CoefT<double> kd;            // fp64 plans
  const void* tab;             // [3][w+2] eta, A, B (T)
  const float* eta;            // stored (user-supplied) eta [nz][ny][pitch] or null
  double dt;
};

template <typename T> __device__ __forceinline__ const CoefT<T>& naive_coef(const NaiveParams& P);
template <> __device__ __forceinline__ const CoefT<float>& naive_coef<float>(const NaiveParams& P) { return P.k; }
template <> __device__ __forceinline__ const CoefT<double>& naive_coef<double>(const NaiveParams& P) { return P.kd; }

// One thread per point; all 25 u loads from global memory (x/y fringe by
// bounds checks, z fringe / halo from the ghost planes).  PML-vs-inner choice
// per point ("single kernel with conditionals").
template <typename T>
__global__ void __launch_bounds__(128) k_naive(const T* __restrict__ u, T* __restrict__ up,
                                               const T* __restrict__ vdt2, const NaiveParams P) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 4 + threadIdx.y;
  const int z = P.z0 + blockIdx.z;
  if (x >= P.nx || y >= P.ny) return;
  const CoefT<T>& K = naive_coef<T>(P);
  auto U = [&](int i, int j, int k) -> T {
    if (i < 0 || i >= P.nx || j < 0 || j >= P.ny) return T(0);
    return u[(int64_t)(k + R) * P.plane + (int64_t)j * P.pitch + i];
  };
  NbrT<T> n;
#pragma unroll
  for (int m = 1; m <= R; ++m) {
    n.xm[m - 1] = U(x - m, y, z); n.xp[m - 1] = U(x + m, y, z);
    n.ym[m - 1] = U(x, y - m, z); n.yp[m - 1] = U(x, y + m, z);
    n.zm[m - 1] = U(x, y, z - m); n.zp[m - 1] = U(x, y, z + m);
  }
  const T uc = U(x, y, z);
  const int64_t o = (int64_t)(z + R) * P.plane + (int64_t)y * P.pitch + x;
  const T upc = up[o];
  const T vc = vdt2[(int64_t)z * P.ny * P.pitch + (int64_t)y * P.pitch + x];
  const T L = lap8(K, uc, n);
  const int kg = z + P.zoff;
  const int dx = dist1(x, P.nx, P.w), dy = dist1(y, P.ny, P.w), dz = dist1(kg, P.nzg, P.w);
  const int d = max(max(dx, dy), dz);
  T res;
  if (d == 0) {
    res = upd_inner(L, uc, upc, vc);
  } else {
    const int TN = P.w + 2;
    const T* eta = static_cast<const T*>(P.tab);
    if (P.eta) {
      // stored eta: the 7-point star from the field, A/B from the point
      auto E = [&](int i, int j, int k) -> T {
        if (i < 0 || i >= P.nx || j < 0 || j >= P.ny || k < 0 || k >= P.nzl) return T(0);
        return (T)__ldg(P.eta + ((int64_t)k * P.ny + j) * P.pitch + i);
      };
      const T g = add_rn(add_rn(gterm(E(x + 1, y, z), E(x - 1, y, z), n.xp[0], n.xm[0], K.i2h[0]),
                                gterm(E(x, y + 1, z), E(x, y - 1, z), n.yp[0], n.ym[0], K.i2h[1])),
                         gterm(E(x, y, z + 1), E(x, y, z - 1), n.zp[0], n.zm[0], K.i2h[2]));
      const double e0 = (double)E(x, y, z);
      res = upd_pml(L, g, uc, upc, vc, (T)(1.0 - e0 * P.dt), (T)(1.0 + e0 * P.dt));
    } else {
    const T exp_ = __ldg(eta + max(max(dist1(x + 1, P.nx, P.w), dy), dz));
    const T exm = __ldg(eta + max(max(dist1(x - 1, P.nx, P.w), dy), dz));
    const T eyp = __ldg(eta + max(max(dx, dist1(y + 1, P.ny, P.w)), dz));
    const T eym = __ldg(eta + max(max(dx, dist1(y - 1, P.ny, P.w)), dz));
    const T ezp = __ldg(eta + max(max(dx, dy), dist1(kg + 1, P.nzg, P.w)));
    const T ezm = __ldg(eta + max(max(dx, dy), dist1(kg - 1, P.nzg, P.w)));
    const T g = add_rn(add_rn(gterm(exp_, exm, n.xp[0], n.xm[0], K.i2h[0]),
                              gterm(eyp, eym, n.yp[0], n.ym[0], K.i2h[1])),
                       gterm(ezp, ezm, n.zp[0], n.zm[0], K.i2h[2]));
    res = upd_pml(L, g, uc, upc, vc, __ldg(eta + TN + d), __ldg(eta + 2 * TN + d));
    }
  }
  up[o] = res;
}

// Source injection, PAPER.md L263 (Alg. 1) / SPEC.md L158-161: u_next[src] +=
// inc[n], n = the device step counter (so replayed CUDA graphs stay correct).
// `mlo` / `mhi` (or null): the same cell in the lower / upper neighbour's
// ghost planes (fused halo exchange), which must carry the injected value too
// (both, on a slab thinner than 2R planes).
template <typename T>
__global__ void k_source(T* __restrict__ buf, int64_t off, const T* __restrict__ inc,
                         int64_t ninc, unsigned long long* __restrict__ dstep, T* mlo, T* mhi) {
  const unsigned long long n = *dstep;
  if (n < (unsigned long long)ninc) {
    const T v = add_rn(buf[off], inc[n]);
    buf[off] = v;
    if (mlo) *mlo = v;
    if (mhi) *mhi = v;
  }
  *dstep = n + 1;
}

// Source into a value computed by a wall kernel of a two-step pair:
// buf[off] += inc[n + delta], n = the device step counter (not advanced).
template <typename T>
__global__ void k_source_at(T* __restrict__ buf, int64_t off, const T* __restrict__ inc, int64_t ninc,
                            const unsigned long long* __restrict__ dstep, int delta) {
  const unsigned long long n = *dstep + (unsigned long long)delta;
  if (n < (unsigned long long)ninc) buf[off] = add_rn(buf[off], inc[n]);
}

// advance the device step counter by `by` (after a two-step pair)
__global__ void k_advance(unsigned long long* dstep, int by) { *dstep += (unsigned long long)by; }

// ---- fused halo exchange: neighbour step flags (system scope) -------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Wait until the neighbours have completed as many steps as this rank.  The
// wait is bounded by `timeout_ns` of device time (%globaltimer): a neighbour
// that is dead or mis-wired sets bit 0 (lower) / bit 1 (upper) of *err and the
// wait gives up -- no trap, so the CUDA context survives; the step's results
// are then invalid and wave_peer_check reports WAVE_ERR_PEER.  Once *err is
// set, later waits return at once (the run is already void).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_peer_wait(const unsigned long long* flags, const unsigned long long* done, int need_lo,
                            int need_hi, unsigned long long* err, unsigned long long timeout_ns) {
  const unsigned long long d = *done;
  if (*err) return;
  const unsigned long long t0 = globaltimer_ns();
  for (int side = 0; side < 2; ++side) {
    if (!(side == 0 ? need_lo : need_hi)) continue;
    while (ld_acquire_sys(flags + side) < d) {
      __nanosleep(256);
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicOr(err, 1ull << side);
        return;
      }
    }
  }
}

// Publish "one more step completed" to both neighbours: [0] of the upper
// neighbour's flags = my count as its lower neighbour, [1] of the lower one's.
__global__ void k_peer_signal(unsigned long long* done, unsigned long long* lo_flags,
                              unsigned long long* hi_flags) {
  const unsigned long long d = *done + 1;
  *done = d;
  __threadfence_system();
  if (lo_flags) st_release_sys(lo_flags + 1, d);
  if (hi_flags) st_release_sys(hi_flags + 0, d);
}

// Copy 4 planes (plane pitch `plane` floats) to a peer buffer.
__global__ void k_copy_planes(const float4* __restrict__ src, float4* dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// vdt2 = (V dt)^2 computed in fp64, rounded once to T (R8), from
// the fp32 V in a padded-pitch buffer (in place for T = float: element by
// element, read before write).
template <typename T>
__global__ void k_vdt2(T* out, const float* V, int64_t pitch, int nx, int64_t rows, double dt) {
  // rows by blocks, x by threads in groups of 4 (pitch is a multiple of 4, rows
  // 16-B aligned): coalesced vector loads, no per-element division
  const int nx4 = (nx + 3) / 4;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x)
    for (int x4 = threadIdx.x; x4 < nx4; x4 += blockDim.x) {
      // the row's last vector may reach into the (never written) pitch padding:
      // load only the valid elements there
      float vv[4] = {0.f, 0.f, 0.f, 0.f};
      if (4 * x4 + 3 < nx) {
        const float4 v = *reinterpret_cast<const float4*>(V + row * pitch + 4 * x4);
        vv[0] = v.x; vv[1] = v.y; vv[2] = v.z; vv[3] = v.w;
      } else {
        for (int c = 0; 4 * x4 + c < nx; ++c) vv[c] = V[row * pitch + 4 * x4 + c];
      }
      T o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double a = (double)vv[c] * dt;
        o[c] = (T)(a * a);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (4 * x4 + c < nx) out[row * pitch + 4 * x4 + c] = o[c];
    }
}

// source increments inc[n] = T(vdt2[src] * w[n]) (the product in fp64: exact
// for fp32 operands)
template <typename T>
__global__ void k_inc(T* __restrict__ inc, const float* __restrict__ wl, int64_t ns, const T* __restrict__ vsrc) {
  const double vs = (double)(*vsrc);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
    inc[i] = (T)(vs * (double)wl[i]);
}

// Exhaustive check of the table division (common.cuh div_table, Markstein's
// reciprocal + FMA correction) against the IEEE division for one plan's B_d:
// every fp32 significand of n in the binades [1, 2) and [2^-80, 2^-79) (the
// smallest |n| the fast path takes) for every d (blockIdx.y).  Negative n
// negates every step exactly (RN is sign-symmetric), and scaling n by 2^k
// scales q0, the residual and q exactly while they stay normal, so these
// binades cover every n the fast path accepts.  mism[0] counts differences.
__global__ void k_divcheck(const float* __restrict__ tab, int T, unsigned* mism) {
  const float B = tab[2 * T + blockIdx.y], rB = tab[3 * T + blockIdx.y];
  unsigned bad = 0;
  for (unsigned m = blockIdx.x * blockDim.x + threadIdx.x; m < (1u << 23); m += gridDim.x * blockDim.x)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float n = __uint_as_float(((k == 0 ? 127u : 47u) << 23) | m);   // 2^0 and 2^-80 binades
      const float a = div_table(n, B, rB, true), b = __fdiv_rn(n, B);
      bad += __float_as_uint(a) != __float_as_uint(b);
    }
  if (bad) atomicAdd(mism, bad);
}

struct Stats {
  unsigned int max_bits;       // max |x| as float bits (finite values only)
  unsigned int min_bits;       // min x as float bits (positive values only)
  unsigned int bad;            // count of non-finite (or non-positive when checking V)
  unsigned int pad;
};

// max|u| / min / non-finite count over a padded-pitch field (max/min
// reported in fp32).
template <typename T>
__global__ void k_stats(const T* __restrict__ buf, int64_t pitch, int nx, int64_t rows,
                        int positive_required, Stats* __restrict__ out) {
  unsigned int mx = 0, mn = 0x7f7fffffu, bad = 0;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x)
  for (int x = threadIdx.x; x < nx; x += blockDim.x) {
    const T vt = buf[row * pitch + x];
    if (!isfinite(vt)) { ++bad; continue; }
    const float v = (float)vt;
    // positive_required: 1 = must be > 0 (velocity), 2 = must be >= 0 (eta)
    if (!isfinite(v) || (positive_required == 1 && !(v > 0.f)) || (positive_required == 2 && !(v >= 0.f))) {
      ++bad;
      continue;
    }
    const unsigned int ab = __float_as_uint(fabsf(v));
    mx = max(mx, ab);
    if (v > 0.f) mn = min(mn, __float_as_uint(v));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out->max_bits, mx);
    atomicMin(&out->min_bits, mn);
    if (bad) atomicAdd(&out->bad, bad);
  }
}

}  // namespace w25
