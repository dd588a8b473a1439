// paper_shapes.cuh -- the paper's GPU code shapes (§III),
// written the paper's way (one point per thread, thread-cooperative loads,
// __syncthreads between phases, no TMA / mbarriers / warp specialisation) for
// the code-shape ablation on B200.  They compute the
// interior column (inner xy footprint x all z, z caps plane-uniform) with the
// same per-point arithmetic as every other kernel (common.cuh), so each is
// bitwise equal to the production k_stream; they are selected only through the
// WAVE25_ABLATION environment variable (never by default).
//
//   gmem_DXxDYxDZ   all 25 loads from global memory
//   smem_u          3-D 8x8x8 tile + star halos in shared memory (L455-489)
//   st_smem_DXxDY   2.5-D streaming, 2R+1 = 9 planes in shared memory (L618-664)
//   st_reg_shft     2.5-D streaming, xy plane in shared memory, z window in 9
//                   registers shifted every plane (L666-717)
//   st_reg_fixed    same with fixed registers and the loop unrolled 9x (L735-775)
//   semi            streaming with the semi-stencil along z (L580-617); not
//                   bitwise (different summation order), within the 1e-5 gate
#pragma once
#include "stream.cuh"

namespace w25 {

struct AblParams {
  const float* u;               // u^n, padded layout base
  const float* up;              // u^{n-1} (the output buffer: read at the centre only)
  float* out;                   // u^{n+1} (= up for the in-place step)
  const float* v;               // vdt2, [nz][ny][pitch]
  int64_t pitch, plane;
  int nx, ny, nzl, nzg, zoff, w;
  int x0, x1, y0, y1, z0, z1;   // region (local z)
  Coef k;
  const float* tab;             // [3][w+2]
};

// CHK: bounds-check x/y (only needed when the region is closer than R to the
// domain edge, i.e. w < R); the paper's inner-region kernels need no checks
template <bool CHK>
__device__ __forceinline__ float abl_u(const AblParams& P, int x, int y, int z) {
  if (CHK && (x < 0 || x >= P.nx || y < 0 || y >= P.ny)) return 0.f;     // Dirichlet fringe
  // L2-only load (ld.global.cg): u^n was written by other kernels of the same
  // CUDA graph (walls on a side branch); an L1 line cached by an earlier
  // kernel on this SM must never be hit
  return __ldcg(P.u + (int64_t)(z + R) * P.plane + (int64_t)y * P.pitch + x);
}

// inner update or the plane-uniform z-cap PML update of one point (x, y inner),
// the arithmetic of cap_update for one component
__device__ __forceinline__ float abl_update(const AblParams& P, int kg, float L, float c, float up, float v,
                                            float xp, float xm, float yp, float ym, float zp, float zm) {
  if (kg >= P.w && kg < P.nzg - P.w) return upd_inner(L, c, up, v);
  const int T = P.w + 2;
  const int dz = dist1(kg, P.nzg, P.w);
  const float ex = __ldg(P.tab + dz), ezp = __ldg(P.tab + dist1(kg + 1, P.nzg, P.w)),
              ezm = __ldg(P.tab + dist1(kg - 1, P.nzg, P.w));
  const float g = __fadd_rn(__fadd_rn(gterm(ex, ex, xp, xm, P.k.i2h[0]), gterm(ex, ex, yp, ym, P.k.i2h[1])),
                            gterm(ezp, ezm, zp, zm, P.k.i2h[2]));
  return upd_pml(L, g, c, up, v, __ldg(P.tab + T + dz), __ldg(P.tab + 2 * T + dz));
}

__device__ __forceinline__ void abl_store(const AblParams& P, int x, int y, int z, float L, float c,
                                          const Nbr& n) {
  const int64_t o = (int64_t)(z + R) * P.plane + (int64_t)y * P.pitch + x;
  const float upc = __ldcg(P.up + o);
  const float vc = __ldcg(P.v + (int64_t)z * P.ny * P.pitch + (int64_t)y * P.pitch + x);
  P.out[o] = abl_update(P, z + P.zoff, L, c, upc, vc, n.xp[0], n.xm[0], n.yp[0], n.ym[0], n.zp[0], n.zm[0]);
}

// ---- gmem_DXxDYxDZ: one thread per point, 25 global loads ------------------
template <int DX, int DY, int DZ, bool CHK>
__global__ void __launch_bounds__(DX * DY * DZ) k_gmem(const AblParams P) {
  const int x = P.x0 + blockIdx.x * DX + threadIdx.x;
  const int y = P.y0 + blockIdx.y * DY + threadIdx.y;
  const int z = P.z0 + blockIdx.z * DZ + threadIdx.z;
  if (x >= P.x1 || y >= P.y1 || z >= P.z1) return;
  Nbr n;
#pragma unroll
  for (int m = 1; m <= R; ++m) {
    n.xm[m - 1] = abl_u<CHK>(P, x - m, y, z); n.xp[m - 1] = abl_u<CHK>(P, x + m, y, z);
    n.ym[m - 1] = abl_u<CHK>(P, x, y - m, z); n.yp[m - 1] = abl_u<CHK>(P, x, y + m, z);
    n.zm[m - 1] = abl_u<CHK>(P, x, y, z - m); n.zp[m - 1] = abl_u<CHK>(P, x, y, z + m);
  }
  const float c = abl_u<CHK>(P, x, y, z);
  abl_store(P, x, y, z, lap8(P.k, c, n), c, n);
}

// ---- smem_u: 8x8x8 block, tile + star halos in shared memory ---------------
// Thread (i, j, k) fetches its point; threads 0..R-1 / R..2R-1 along each
// dimension fetch the halo on one / the other side.
template <bool CHK>
__global__ void __launch_bounds__(512) k_smem_u(const AblParams P) {
  constexpr int D = 8, E = D + 2 * R;
  __shared__ float t[E][E][E];                 // [z][y][x], corners unused
  const int tx = threadIdx.x, ty = threadIdx.y, tz = threadIdx.z;
  const int x = P.x0 + blockIdx.x * D + tx, y = P.y0 + blockIdx.y * D + ty, z = P.z0 + blockIdx.z * D + tz;
  const int xb = P.x0 + blockIdx.x * D, yb = P.y0 + blockIdx.y * D, zb = P.z0 + blockIdx.z * D;
  // z may run past the slab into the ghost planes (zero-filled, valid memory) only up to 4
  auto ld = [&](int xx, int yy, int zz) { return zz >= -R && zz < P.nzl + R ? abl_u<CHK>(P, xx, yy, zz) : 0.f; };
  t[tz + R][ty + R][tx + R] = ld(x, y, z);
  const int hx = tx < R ? xb - R + tx : xb + D + tx - R;
  t[tz + R][ty + R][tx < R ? tx : tx + D] = ld(hx, y, z);
  const int hy = ty < R ? yb - R + ty : yb + D + ty - R;
  t[tz + R][ty < R ? ty : ty + D][tx + R] = ld(x, hy, z);
  const int hz = tz < R ? zb - R + tz : zb + D + tz - R;
  t[tz < R ? tz : tz + D][ty + R][tx + R] = ld(x, y, hz);
  __syncthreads();
  if (x >= P.x1 || y >= P.y1 || z >= P.z1) return;
  Nbr n;
#pragma unroll
  for (int m = 1; m <= R; ++m) {
    n.xm[m - 1] = t[tz + R][ty + R][tx + R - m]; n.xp[m - 1] = t[tz + R][ty + R][tx + R + m];
    n.ym[m - 1] = t[tz + R][ty + R - m][tx + R]; n.yp[m - 1] = t[tz + R][ty + R + m][tx + R];
    n.zm[m - 1] = t[tz + R - m][ty + R][tx + R]; n.zp[m - 1] = t[tz + R + m][ty + R][tx + R];
  }
  const float c = t[tz + R][ty + R][tx + R];
  abl_store(P, x, y, z, lap8(P.k, c, n), c, n);
}

// ---- 2.5-D streaming shapes --------------------------------------------
enum { ST_SMEM = 0, ST_SHFT = 1, ST_FIXED = 2 };

// Load plane z of the (DX+2R) x (DY+2R) star window into `pl` (row stride DX+2R):
// the thread's own point, and the halos by the first 2R threads of each dimension.
template <int DX, int DY, bool CHK>
__device__ __forceinline__ void st_load_plane(const AblParams& P, float* pl, int xb, int yb, int z, int tx,
                                              int ty, bool own, float ownv) {
  constexpr int W = DX + 2 * R;
  const int x = xb + tx, y = yb + ty;
  pl[(ty + R) * W + tx + R] = own ? ownv : abl_u<CHK>(P, x, y, z);
  if (tx < 2 * R) {
    const int hx = tx < R ? xb - R + tx : xb + DX + tx - R;
    pl[(ty + R) * W + (tx < R ? tx : tx + DX)] = abl_u<CHK>(P, hx, y, z);
  }
  if (ty < 2 * R) {
    const int hy = ty < R ? yb - R + ty : yb + DY + ty - R;
    pl[(ty < R ? ty : ty + DY) * W + tx + R] = abl_u<CHK>(P, x, hy, z);
  }
}

template <int SHAPE, int DX, int DY, bool CHK>
__global__ void __launch_bounds__(DX * DY) k_st(const AblParams P) {
  static_assert(DX >= 2 * R && DY >= 2 * R, "the first 2R threads fetch the halos");
  constexpr int W = DX + 2 * R, H = DY + 2 * R, PL = W * H;
  constexpr int NPL = SHAPE == ST_SMEM ? 2 * R + 1 : 1;
  __shared__ float B[NPL * PL];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int xb = P.x0 + blockIdx.x * DX, yb = P.y0 + blockIdx.y * DY;
  const int x = xb + tx, y = yb + ty;
  const bool act = x < P.x1 && y < P.y1;
  const int o = (ty + R) * W + tx + R;
  if (SHAPE == ST_SMEM) {
    // B[0..R): planes z0-4..z0-1, B[R..2R): planes z0..z0+3
    for (int i = 0; i < 2 * R; ++i) st_load_plane<DX, DY, CHK>(P, B + i * PL, xb, yb, P.z0 - R + i, tx, ty, false, 0.f);
#pragma unroll 1
    for (int z0 = P.z0; z0 < P.z1; z0 += 2 * R + 1) {
#pragma unroll
      for (int s = 0; s < 2 * R + 1; ++s) {     // index rotation by unrolling (no modulus)
        const int z = z0 + s;
        if (z >= P.z1) break;
        st_load_plane<DX, DY, CHK>(P, B + ((s + 2 * R) % (2 * R + 1)) * PL, xb, yb, z + R, tx, ty, false, 0.f);
        __syncthreads();
        if (act) {
          const float* c0 = B + ((s + R) % (2 * R + 1)) * PL + o;
          Nbr n;
#pragma unroll
          for (int m = 1; m <= R; ++m) {
            n.xm[m - 1] = c0[-m]; n.xp[m - 1] = c0[m];
            n.ym[m - 1] = c0[-m * W]; n.yp[m - 1] = c0[m * W];
            n.zm[m - 1] = B[((s + R - m + 2 * R + 1) % (2 * R + 1)) * PL + o];
            n.zp[m - 1] = B[((s + R + m) % (2 * R + 1)) * PL + o];
          }
          abl_store(P, x, y, z, lap8(P.k, *c0, n), *c0, n);
        }
        __syncthreads();
      }
    }
  } else {
    // z window in 9 registers: r[0] = z-4 ... r[8] = z+4
    float r[2 * R + 1];
#pragma unroll
    for (int i = 0; i < 2 * R; ++i) r[i] = abl_u<CHK>(P, x, y, P.z0 - R + i);   // also off-region: halo source
    if (SHAPE == ST_SHFT) {
#pragma unroll 1
      for (int z = P.z0; z < P.z1; ++z) {
        r[2 * R] = abl_u<CHK>(P, x, y, z + R);                        // leading point
        st_load_plane<DX, DY, CHK>(P, B, xb, yb, z, tx, ty, true, r[R]);
        __syncthreads();
        if (act) {
          Nbr n;
#pragma unroll
          for (int m = 1; m <= R; ++m) {
            n.xm[m - 1] = B[o - m]; n.xp[m - 1] = B[o + m];
            n.ym[m - 1] = B[o - m * W]; n.yp[m - 1] = B[o + m * W];
            n.zm[m - 1] = r[R - m]; n.zp[m - 1] = r[R + m];
          }
          abl_store(P, x, y, z, lap8(P.k, r[R], n), r[R], n);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 2 * R; ++i) r[i] = r[i + 1];        // shift
      }
    } else {
#pragma unroll 1
      for (int z0 = P.z0; z0 < P.z1; z0 += 2 * R + 1) {
#pragma unroll
        for (int s = 0; s < 2 * R + 1; ++s) {   // fixed registers, rotation by unrolling
          const int z = z0 + s;
          if (z >= P.z1) break;
          r[(s + 2 * R) % (2 * R + 1)] = abl_u<CHK>(P, x, y, z + R);
          const float cur = r[(s + R) % (2 * R + 1)];
          st_load_plane<DX, DY, CHK>(P, B, xb, yb, z, tx, ty, true, cur);
          __syncthreads();
          if (act) {
            Nbr n;
#pragma unroll
            for (int m = 1; m <= R; ++m) {
              n.xm[m - 1] = B[o - m]; n.xp[m - 1] = B[o + m];
              n.ym[m - 1] = B[o - m * W]; n.yp[m - 1] = B[o + m * W];
              n.zm[m - 1] = r[(s + R - m + 2 * R + 1) % (2 * R + 1)];
              n.zp[m - 1] = r[(s + R + m) % (2 * R + 1)];
            }
            abl_store(P, x, y, z, lap8(P.k, cur, n), cur, n);
          }
          __syncthreads();
        }
      }
    }
  }
}

// ---- semi: 2.5-D streaming with the semi-stencil along z (PAPER.md L580-617,
// after de la Cruz et al.).  Every plane value, as soon as it is loaded,
// scatters its z contributions c_zm u(q) into the partial sums of the 2R points
// q-R..q-1 and q+1..q+R it belongs to; the x/y part of point q is added when
// plane q is in shared memory; point q-R is complete.  One load per plane, a
// 2R+1-slot ring of partial sums instead of values.  The summation order
// differs from Eq. 3's (forward/backward halves), so this shape is compared
// with the oracle within the 1e-5 gate, not bitwise.
template <int DX, int DY, bool CHK>
__global__ void __launch_bounds__(DX * DY) k_semi(const AblParams P) {
  constexpr int W = DX + 2 * R, NS = 2 * R + 1;
  __shared__ float B[W * (DY + 2 * R)];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int xb = P.x0 + blockIdx.x * DX, yb = P.y0 + blockIdx.y * DY;
  const int x = xb + tx, y = yb + ty;
  const bool act = x < P.x1 && y < P.y1;
  const int o = (ty + R) * W + tx + R;
  float A[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) A[i] = 0.f;
  // slot of plane p: (p - (z0 - R)) % NS; iteration q runs from z0-R to z1+R-1
#pragma unroll 1
  for (int q0 = P.z0 - R; q0 < P.z1 + R; q0 += NS) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int q = q0 + s;
      if (q >= P.z1 + R) break;
      const float val = abl_u<CHK>(P, x, y, q);
      const bool inq = q >= P.z0 && q < P.z1;          // block-uniform
      if (inq) {
        st_load_plane<DX, DY, CHK>(P, B, xb, yb, q, tx, ty, true, val);
        __syncthreads();
        float xy = __fmul_rn(P.k.c0, val);
#pragma unroll
        for (int m = 1; m <= R; ++m) xy = __fmaf_rn(P.k.cx[m - 1], __fadd_rn(B[o + m], B[o - m]), xy);
#pragma unroll
        for (int m = 1; m <= R; ++m) xy = __fmaf_rn(P.k.cy[m - 1], __fadd_rn(B[o + m * W], B[o - m * W]), xy);
        A[s] = __fadd_rn(A[s], xy);
        __syncthreads();
      }
      // scatter u(q) into the partial sums of q-m (forward half) and q+m (backward half)
#pragma unroll
      for (int m = 1; m <= R; ++m) {
        A[(s - m + NS) % NS] = __fmaf_rn(P.k.cz[m - 1], val, A[(s - m + NS) % NS]);
        A[(s + m) % NS] = __fmaf_rn(P.k.cz[m - 1], val, A[(s + m) % NS]);
      }
      // point p = q - R is complete
      const int p = q - R;
      const int sp = (s - R + NS) % NS;
      if (act && p >= P.z0 && p < P.z1) {
        Nbr n;
        const float c = abl_u<CHK>(P, x, y, p);
        n.xp[0] = abl_u<CHK>(P, x + 1, y, p); n.xm[0] = abl_u<CHK>(P, x - 1, y, p);
        n.yp[0] = abl_u<CHK>(P, x, y + 1, p); n.ym[0] = abl_u<CHK>(P, x, y - 1, p);
        n.zp[0] = abl_u<CHK>(P, x, y, p + 1); n.zm[0] = abl_u<CHK>(P, x, y, p - 1);
        abl_store(P, x, y, p, A[sp], c, n);
      }
      A[sp] = 0.f;                                      // slot reused by plane q + R + 1
    }
  }
}

}  // namespace w25
