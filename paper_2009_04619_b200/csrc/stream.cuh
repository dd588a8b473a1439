// stream.cuh -- the z-streaming stencil kernel for sm_100a (interior column
// and PML walls).  Design:
//
//  * Work unit = one TX x TY xy-tile of one region x one z-chunk [zs, ze).
//    Blocks are ordered chunk-major (all tiles of chunk 0, then chunk 1, ...)
//    so co-resident CTAs are xy-neighbours at similar z and the 4-cell halo
//    rows they re-read come from L2, not HBM.
//  * u planes (tile + 4-cell halo, (TX+8) x (TY+8) floats) arrive by TMA
//    (cp.async.bulk.tensor.3d) into an SU-stage shared-memory ring, one
//    mbarrier per stage.  Out-of-bounds x/y cells are zero-filled by TMA, so
//    the Dirichlet fringe costs nothing.  u_prev and vdt2 planes (tile only)
//    arrive the same way into an SP-stage ring.  Thread 0 refills the stage
//    freed by the plane just finished after one __syncthreads per plane.
//  * Each thread owns 4 consecutive x points (one float4) x TYT rows and keeps
//    the 9 z-planes u(z-4..z+4) of its points in a register queue with fixed
//    slots (slot = plane mod 9, loop unrolled 9x so every slot index is a
//    compile-time constant) -- the paper's st_reg_fixed idea (PAPER.md
//    L735-775).  x neighbours come from 2 LDS.128 per row (left/right float4),
//    y neighbours from 8 LDS.128 per thread-row group, z neighbours from
//    registers.
//  * MODE_INNER: region = inner xy footprint; planes inside the inner z range
//    take the inner update (no per-point branches); the z-PML caps (global
//    planes k < w or k >= nz-w) take the PML update with plane-uniform eta
//    (one warp-uniform branch per plane).  MODE_WALL: x/y PML walls, every
//    point takes the PML update with eta on the 7-point star evaluated from
//    integer distances (no stored eta array, 0 HBM bytes).
#pragma once
#include "common.cuh"

namespace w25 {

enum { MODE_INNER = 0, MODE_WALL = 1 };

struct Region {
  int x0, x1, y0, y1, z0, z1;   // point box [x0,x1) x [y0,y1) x [z0,z1) (local z)
  int ax0;                      // x0 rounded down to a multiple of 4 (tile origin)
  int ntx, nty, nzc;            // tiles in x, y and z-chunks
  int blk0;                     // first blockIdx.x of this region
};

constexpr int MAX_REGIONS = 4;

struct StreamParams {
  float* out;                   // u_next buffer (= u_prev buffer), padded layout base
  int64_t pitch, plane;         // row / plane pitch in floats
  int nx, ny, nzl, nzg, zoff, w;
  int cz;                       // z-chunk length
  int nreg;
  Region reg[MAX_REGIONS];
  Coef k;
  const float* tab;             // [3][w+2]: eta_d, A_d, B_d (d = 0..w), eta_{w+1} = 0
};

template <int TX, int TY, int TYT, int SU, int SP>
struct StreamCfg {
  static constexpr int LX = TX / 4;               // float4 lanes across x
  static constexpr int LY = TY / TYT;             // thread rows
  static constexpr int NT = LX * LY;              // threads per CTA
  static constexpr int SW = TX + 2 * R;           // smem u row stride (floats)
  static constexpr int SH = TY + 2 * R;
  static constexpr int U_STAGE = SW * SH;         // floats per u stage
  static constexpr int P_STAGE = TX * TY;         // floats per u_prev / vdt2 stage
  static constexpr int BAR_OFF = (SU * U_STAGE + 2 * SP * P_STAGE) * 4;  // bytes
  static constexpr int TAB_OFF = BAR_OFF + (SU + SP) * 8;
  static size_t smem_bytes(int w) { return TAB_OFF + 3 * (w + 2) * 4; }
  static_assert(TX % 4 == 0 && TY % TYT == 0, "tile shape");
  static_assert((U_STAGE * 4) % 128 == 0 && (P_STAGE * 4) % 128 == 0, "TMA smem alignment");
  static_assert(SU >= 8, "u ring must hold the 8 warm-up planes");
  static_assert(NT % 32 == 0, "whole warps");
};

template <int TX, int TY, int TYT, int SU, int SP, int MODE>
__global__ void __launch_bounds__(StreamCfg<TX, TY, TYT, SU, SP>::NT)
k_stream(const __grid_constant__ CUtensorMap tm_u,    // u^n, box (TX+8, TY+8, 1)
         const __grid_constant__ CUtensorMap tm_up,   // u^{n-1}, box (TX, TY, 1)
         const __grid_constant__ CUtensorMap tm_v,    // vdt2, box (TX, TY, 1)
         const StreamParams P) {
  using C = StreamCfg<TX, TY, TYT, SU, SP>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* su = reinterpret_cast<float*>(smem_raw);
  float* sup = su + SU * C::U_STAGE;
  float* sv = sup + SP * C::P_STAGE;
  uint64_t* bar_u = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
  uint64_t* bar_p = bar_u + SU;
  float* stab = reinterpret_cast<float*>(smem_raw + C::TAB_OFF);
  const int TABN = P.w + 2;

  // ---- work unit ---------------------------------------------------------
  int b = blockIdx.x, ri = 0;
#pragma unroll 1
  while (ri + 1 < P.nreg && b >= P.reg[ri + 1].blk0) ++ri;
  const Region G = P.reg[ri];
  b -= G.blk0;
  const int ncol = G.ntx * G.nty;
  const int zc = b / ncol;
  const int rem = b - zc * ncol;
  const int tyi = rem / G.ntx;
  const int txi = rem - tyi * G.ntx;
  const int tx0 = G.ax0 + txi * TX;
  const int ty0 = G.y0 + tyi * TY;
  const int zs = G.z0 + zc * P.cz;
  const int ze = min(zs + P.cz, G.z1);

  const int tid = threadIdx.x;
  const int lx = tid % C::LX;
  const int ly = tid / C::LX;
  const int gx = tx0 + 4 * lx;              // first x of my float4
  const int gy = ty0 + ly * TYT;            // first y of my rows
  const int scol = 4 * lx + R;              // smem column of my float4
  const int srow0 = ly * TYT + R;           // smem row of my first row

  // ---- setup: barriers, PML tables, prologue TMA ------------------------
  if (tid == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_up);
    prefetch_tmap(&tm_v);
    for (int s = 0; s < SU; ++s) mbar_init(&bar_u[s], 1);
    for (int s = 0; s < SP; ++s) mbar_init(&bar_p[s], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < 3 * TABN; i += C::NT) stab[i] = P.tab[i];
  __syncthreads();

  const uint64_t pol_u = policy_evict_last();    // u^n: re-read (halo) by neighbours
  const uint64_t pol_s = policy_evict_first();   // u^{n-1}, vdt2: streamed once
  auto issue_u = [&](int p) {                     // plane p (local z), p >= zs-4
    const int s = (p - zs + R) % SU;
    mbar_arrive_expect_tx(&bar_u[s], C::U_STAGE * 4);
    tma_load_3d(su + s * C::U_STAGE, &tm_u, &bar_u[s], tx0 - R, ty0 - R, p + R, pol_u);
  };
  auto issue_p = [&](int p) {
    const int s = (p - zs) % SP;
    mbar_arrive_expect_tx(&bar_p[s], 2 * C::P_STAGE * 4);
    tma_load_3d(sup + s * C::P_STAGE, &tm_up, &bar_p[s], tx0, ty0, p + R, pol_s);
    tma_load_3d(sv + s * C::P_STAGE, &tm_v, &bar_p[s], tx0, ty0, p, pol_s);
  };
  if (tid == 0) {
    for (int p = zs - R; p < zs - R + SU && p <= ze + R - 1; ++p) issue_u(p);
    for (int p = zs; p < zs + SP && p < ze; ++p) issue_p(p);
  }

  // ---- per-thread geometry: store mask, PML distances --------------------
  unsigned mask = 0;                         // bit (r*4 + c): point is in the region
#pragma unroll
  for (int r = 0; r < TYT; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int x = gx + c, y = gy + r;
      if (x >= G.x0 && x < G.x1 && y >= G.y0 && y < G.y1) mask |= 1u << (r * 4 + c);
    }
  const bool full = mask == (TYT * 4 == 32 ? 0xffffffffu : ((1u << (TYT * 4)) - 1u));
  int dxs[6], dys[TYT + 2];                  // distances at x = gx-1..gx+4, y = gy-1..gy+TYT
  if (MODE == MODE_WALL) {
#pragma unroll
    for (int c = 0; c < 6; ++c) dxs[c] = dist1(gx - 1 + c, P.nx, P.w);
#pragma unroll
    for (int r = 0; r < TYT + 2; ++r) dys[r] = dist1(gy - 1 + r, P.ny, P.w);
  }
  float* outp = P.out + (int64_t)gy * P.pitch + gx;

  // ---- warm-up: planes zs-4 .. zs+3 into queue slots 0..7 ----------------
  float4 q[9][TYT];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int p = zs - R + s;
    const int st = (p - zs + R) % SU;
    mbar_wait(&bar_u[st], ((p - zs + R) / SU) & 1);
#pragma unroll
    for (int r = 0; r < TYT; ++r)
      q[s][r] = lds4(su + st * C::U_STAGE + (srow0 + r) * C::SW + scol);
  }
  __syncthreads();                           // stages of planes zs-4..zs-1 are free
  if (tid == 0) {
    fence_proxy_async_smem();
    for (int p = zs - R + SU; p < zs + SU; ++p)
      if (p <= ze + R - 1) issue_u(p);
  }

  const Coef& K = P.k;
  // ---- main loop over planes, unrolled 9x (fixed register slots) ---------
#pragma unroll 1
  for (int z0 = zs; z0 < ze; z0 += 9) {
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int z = z0 + s;
      if (z >= ze) break;
      // slot of plane z+o is (s + 4 + o) mod 9 (compile-time)
      // 1. leading plane z+4 -> queue
      {
        const int p = z + R;
        const int st = (p - zs + R) % SU;
        mbar_wait(&bar_u[st], ((p - zs + R) / SU) & 1);
#pragma unroll
        for (int r = 0; r < TYT; ++r)
          q[(s + 8) % 9][r] = lds4(su + st * C::U_STAGE + (srow0 + r) * C::SW + scol);
      }
      // 2. u^{n-1} and vdt2 of plane z
      float4 upv[TYT], vv[TYT];
      {
        const int st = (z - zs) % SP;
        mbar_wait(&bar_p[st], ((z - zs) / SP) & 1);
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          upv[r] = lds4(sup + st * C::P_STAGE + (ly * TYT + r) * TX + 4 * lx);
          vv[r] = lds4(sv + st * C::P_STAGE + (ly * TYT + r) * TX + 4 * lx);
        }
      }
      // 3. compute plane z from the u stage of plane z
      const float* S = su + ((z - zs + R) % SU) * C::U_STAGE;
      float4 Y[TYT + 2 * R];                 // rows gy-4 .. gy+TYT+3 at my float4
#pragma unroll
      for (int j = 0; j < TYT + 2 * R; ++j) {
        if (j >= R && j < R + TYT) Y[j] = q[(s + 4) % 9][j - R];
        else Y[j] = lds4(S + (srow0 - R + j) * C::SW + scol);
      }
      const int kg = z + P.zoff;
      bool pml_plane = false;
      float A_c = 1.f, B_c = 1.f, ez_p = 0.f, ez_m = 0.f, ex_c = 0.f;
      int dzk = 0, dzp = 0, dzm = 0;
      if (MODE == MODE_INNER) {
        pml_plane = (kg < P.w) || (kg >= P.nzg - P.w);
        if (pml_plane) {
          dzk = dist1(kg, P.nzg, P.w);
          A_c = stab[TABN + dzk];
          B_c = stab[2 * TABN + dzk];
          ex_c = stab[dzk];
          ez_p = stab[dist1(kg + 1, P.nzg, P.w)];
          ez_m = stab[dist1(kg - 1, P.nzg, P.w)];
        }
      } else {
        dzk = dist1(kg, P.nzg, P.w);
        dzp = dist1(kg + 1, P.nzg, P.w);
        dzm = dist1(kg - 1, P.nzg, P.w);
      }
#pragma unroll
      for (int r = 0; r < TYT; ++r) {
        const float* Srow = S + (srow0 + r) * C::SW + scol;
        const float4 Lf = lds4(Srow - 4);
        const float4 Ce = Y[R + r];
        const float4 Rf = lds4(Srow + 4);
        const float X[12] = {Lf.x, Lf.y, Lf.z, Lf.w, Ce.x, Ce.y, Ce.z, Ce.w, Rf.x, Rf.y, Rf.z, Rf.w};
        float res[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          Nbr n;
#pragma unroll
          for (int m = 1; m <= R; ++m) {
            n.xm[m - 1] = X[4 + c - m];
            n.xp[m - 1] = X[4 + c + m];
            n.ym[m - 1] = f4get(Y[R + r - m], c);
            n.yp[m - 1] = f4get(Y[R + r + m], c);
            n.zm[m - 1] = f4get(q[(s + 4 - m + 9) % 9][r], c);
            n.zp[m - 1] = f4get(q[(s + 4 + m) % 9][r], c);
          }
          const float uc = X[4 + c];
          const float L = lap8(K, uc, n);
          const float upc = f4get(upv[r], c), vc = f4get(vv[r], c);
          if (MODE == MODE_INNER) {
            if (!pml_plane) {
              res[c] = upd_inner(L, uc, upc, vc);
            } else {
              // inner xy footprint inside a z cap: eta(x +- 1) = eta(y +- 1) = eta_dz
              const float g = __fadd_rn(__fadd_rn(gterm(ex_c, ex_c, n.xp[0], n.xm[0], K.i2h[0]),
                                                  gterm(ex_c, ex_c, n.yp[0], n.ym[0], K.i2h[1])),
                                        gterm(ez_p, ez_m, n.zp[0], n.zm[0], K.i2h[2]));
              res[c] = upd_pml(L, g, uc, upc, vc, A_c, B_c);
            }
          } else {
            const int dxc = dxs[c + 1], dyc = dys[r + 1];
            const int dxy = max(dxc, dyc);
            const int d = max(dxy, dzk);
            const float exp_ = stab[max(max(dxs[c + 2], dyc), dzk)];
            const float exm = stab[max(max(dxs[c], dyc), dzk)];
            const float eyp = stab[max(max(dxc, dys[r + 2]), dzk)];
            const float eym = stab[max(max(dxc, dys[r]), dzk)];
            const float ezp = stab[max(dxy, dzp)];
            const float ezm = stab[max(dxy, dzm)];
            const float g = __fadd_rn(__fadd_rn(gterm(exp_, exm, n.xp[0], n.xm[0], K.i2h[0]),
                                                gterm(eyp, eym, n.yp[0], n.ym[0], K.i2h[1])),
                                      gterm(ezp, ezm, n.zp[0], n.zm[0], K.i2h[2]));
            res[c] = upd_pml(L, g, uc, upc, vc, stab[TABN + d], stab[2 * TABN + d]);
          }
        }
        // 4. store u_next (streaming; masked on ragged tiles)
        float* o = outp + (int64_t)(z + R) * P.plane + (int64_t)r * P.pitch;
        if (full) {
          st_cs_f4(o, make_float4(res[0], res[1], res[2], res[3]));
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (mask & (1u << (r * 4 + c))) o[c] = res[c];
        }
      }
      // 5. release the stages of plane z, refill them
      __syncthreads();
      if (tid == 0) {
        fence_proxy_async_smem();
        if (z + SU <= ze + R - 1) issue_u(z + SU);
        if (z + SP < ze) issue_p(z + SP);
      }
    }
  }
}

}  // namespace w25
