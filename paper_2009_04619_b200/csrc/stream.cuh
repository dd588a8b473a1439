// stream.cuh -- the z-streaming stencil kernel for sm_100a (interior column
// and PML walls).  Design:
//
//  * Work unit = one CW x TY xy-tile (CW = computed width) of one region x one
//    z-chunk [zs, ze).  Blocks are ordered chunk-major (all tiles of chunk 0,
//    then chunk 1, ...) so co-resident CTAs are xy-neighbours at similar z and
//    the 4-cell halo rows they re-read come from L2, not HBM.
//  * A producer warp streams, by TMA (cp.async.bulk.tensor.3d), u planes of a
//    TX-wide box + 4-cell halo ((TX+8) x (TY+8) floats, TX >= CW, 128-B
//    aligned where possible) into a 9-stage shared-memory ring and u_prev /
//    vdt2 tiles (CW x TY) into a 3-stage ring; full/empty mbarrier pairs per
//    stage (Blackwell producer/consumer pipeline, no block-wide barrier in the
//    loop).  Out-of-bounds x/y cells are zero-filled by TMA, so the Dirichlet
//    fringe costs nothing.  An L2 tensor prefetch runs P.pf planes ahead.
//    9 = the z-window 2R+1, so with the plane loop unrolled 9x every stage
//    index, register-queue slot and mbarrier parity is a compile-time constant.
//  * Each consumer thread owns 4 consecutive x points (one float4) x TYT rows
//    and keeps u(z-4..z+4) of its points in a 9-slot register queue with fixed
//    slots -- the paper's st_reg_fixed idea.  x neighbours:
//    2 LDS.128 per row; y neighbours: 8 LDS.128 per thread; z: registers.
//  * All 4*TYT points of a plane are evaluated as interleaved independent FMA
//    chains; the PML-vs-inner choice is one uniform branch per plane.
//  * MODE_INNER: region = inner xy footprint over all z; planes inside the
//    inner z range take the inner update (no per-point branches); the z-PML
//    caps (global k < w or k >= nz-w) take the PML update with plane-uniform
//    eta through a non-inlined function (keeps the hot loop's code small).
//  * MODE_WALL: the x walls (left/right) and y walls (front/back) over all z;
//    every point takes the PML update.  eta on the 7-point star is evaluated
//    from integer distances (no stored eta array, 0 extra HBM bytes); its
//    z-invariant part (grad-eta coefficients, A, B) is precomputed per point
//    once, and only the planes next to the z caps re-evaluate it in full.
#pragma once
#include "common.cuh"

namespace w25 {

// MODE_FUSED: whole xy plane in one launch, path chosen per warp and plane.
// MODE_NULL: memory-pattern probe (no stencil; wrong results, diagnostics only).
enum { MODE_INNER = 0, MODE_WALL = 1, MODE_NULL = 2, MODE_FUSED = 3 };

struct Region {
  int x0, x1, y0, y1, z0, z1;   // point box [x0,x1) x [y0,y1) x [z0,z1) (local z)
  int ax0;                      // x0 rounded down to a multiple of 4 (first computed column)
  int ntx, nty, nzc;            // tiles in x (step CW), y (step TY) and z-chunks
  int blk0;                     // first blockIdx.x of this region
};

constexpr int MAX_REGIONS = 4;
constexpr int SU = 9;           // u ring stages  (= 2R+1)
constexpr int SP = 3;           // u_prev/vdt2 ring stages (divides 9)

struct StreamParams {
  float* out;                   // u_next buffer (= u_prev buffer), padded layout base
  float* rlo;                   // lower neighbour's upper ghost planes (next buffer) or null
  float* rhi;                   // upper neighbour's lower ghost planes (next buffer) or null
  int64_t pitch, plane;         // row / plane pitch in floats
  int nx, ny, nzl, nzg, zoff, w;
  int cz;                       // z-chunk length
  int pf;                       // L2 prefetch distance (planes beyond the rings; 0 = off)
  int order;                    // tile order in a chunk: 0 = x fastest; G > 0 = groups of G x-tiles, y inside
  int upol;                     // L2 policy of u loads: 0 = evict_last, 1 = evict_normal
  int nreg;
  Region reg[MAX_REGIONS];
  Coef k;
  const float* tab;             // [3][w+2]: eta_d, A_d, B_d (d = 0..w), eta_{w+1} = 0
};

// RA > 0: one CTA per SM with a producer WARPGROUP (4 warps, one issuing TMA)
// that gives its registers back (setmaxnreg.dec to 24) so that the consumer
// warpgroups can raise theirs to RA (setmaxnreg.inc) -- Blackwell/Hopper
// warp-specialised register reallocation.  Needs NWC % 4 == 0.
template <int TX, int CW, int TY, int TYT, int MINB = 2, int RA = 0>
struct StreamCfg {
  static constexpr int LXW = (CW / 4) < 8 ? (CW / 4) : 8;   // float4 lanes per warp row
  static constexpr int LYW = 32 / LXW;                      // thread rows per warp
  static constexpr int WX = (CW / 4 + LXW - 1) / LXW;      // consumer warps across x (the last
                                                            // may have idle "phantom" lanes)
  static constexpr int WY = (TY / TYT) / LYW;               // consumer warps in y
  static constexpr int NWC = WX * WY;                       // consumer warps
  static constexpr int NPW = RA > 0 ? 4 : 1;                // producer warps
  static constexpr int NT = 32 * (NWC + NPW);
  // register cap for MINB CTAs per SM: warps are placed round-robin on the 4
  // sub-partitions, each with a 16K-register file
  static constexpr int WPS = (MINB * (NWC + NPW) + 3) / 4;  // warps per sub-partition
  static constexpr int MAXR_ = (16384 / (32 * WPS)) & ~7;
  static constexpr int MAXR = MAXR_ > 255 ? 255 : MAXR_;
  static constexpr int SW = TX + 2 * R;                     // smem u row stride (floats)
  static constexpr int SH = TY + 2 * R;
  static constexpr int U_STAGE = SW * SH;                   // floats per u stage
  static constexpr int P_STAGE = CW * TY;                   // floats per u_prev / vdt2 stage
  static constexpr int BAR_OFF = (SU * U_STAGE + 2 * SP * P_STAGE) * 4;  // bytes
  static constexpr int TAB_OFF = BAR_OFF + 2 * (SU + SP) * 8;
  static size_t smem_bytes(int w) { return TAB_OFF + 3 * (w + 2) * 4; }
  static_assert(CW % 4 == 0 && CW <= TX && TX % 4 == 0, "tile widths");
  static_assert(32 % LXW == 0 && (TY / TYT) % LYW == 0 && TY % TYT == 0, "warp tiling");
  static_assert((U_STAGE * 4) % 128 == 0 && (P_STAGE * 4) % 128 == 0, "TMA smem alignment");
  static_assert(RA == 0 || (MINB == 1 && NWC % 4 == 0 && RA % 8 == 0 &&
                            NWC / 4 * RA + 24 <= (NWC / 4 + 1) * MAXR), "register reallocation budget");
};

struct PmlGeo { int nx, ny, nzg, w, T; float i2hx, i2hy, i2hz; };

// Plane-uniform constants of a z-PML cap plane seen from the inner xy footprint.
struct CapC { float ex, ezp, ezm, A, B; };

// PML update of one float4 row inside a z cap (inner x,y => eta(x+-1) =
// eta(y+-1) = eta_dz); same arithmetic as the naive kernel's PML branch.
__device__ __noinline__ float4 cap_update(float4 L, float4 C, float4 up, float4 v, float4 xp, float4 xm,
                                          float4 yp, float4 ym, float4 zp, float4 zm, CapC cc,
                                          float i2hx, float i2hy, float i2hz) {
  float res[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float g = __fadd_rn(__fadd_rn(gterm(cc.ex, cc.ex, f4get(xp, c), f4get(xm, c), i2hx),
                                        gterm(cc.ex, cc.ex, f4get(yp, c), f4get(ym, c), i2hy)),
                              gterm(cc.ezp, cc.ezm, f4get(zp, c), f4get(zm, c), i2hz));
    res[c] = upd_pml(f4get(L, c), g, f4get(C, c), f4get(up, c), f4get(v, c), cc.A, cc.B);
  }
  return make_float4(res[0], res[1], res[2], res[3]);
}

// PML path for one float4 row (4 x-points at gx.., row gy, global plane kg):
// per point the Chebyshev distance d, eta on the 7-point star from the
// (w+2)-entry table (eta_{w+1} = 0 outside), the grad-eta . grad-u term and
// the damped update; points with d = 0 take the inner formula (identical
// arithmetic to the naive kernel).  Used for wall planes in / next to a cap.
__device__ __noinline__ float4 pml_row_call(float4 L, float4 C, float4 up, float4 v, float4 xp, float4 xm,
                                            float4 yp, float4 ym, float4 zp, float4 zm, int gx, int gy, int kg,
                                            PmlGeo G, const float* stab) {
  const int dy = dist1(gy, G.ny, G.w), dyp = dist1(gy + 1, G.ny, G.w), dym = dist1(gy - 1, G.ny, G.w);
  const int dz = dist1(kg, G.nzg, G.w), dzp = dist1(kg + 1, G.nzg, G.w), dzm = dist1(kg - 1, G.nzg, G.w);
  int dxs[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) dxs[c] = dist1(gx - 1 + c, G.nx, G.w);
  float res[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int dx = dxs[c + 1];
    const int dxy = max(dx, dy);
    const int d = max(dxy, dz);
    const float uc = f4get(C, c), upc = f4get(up, c), vc = f4get(v, c);
    const float Lc = f4get(L, c);
    if (d == 0) {
      res[c] = upd_inner(Lc, uc, upc, vc);
    } else {
      const float exp_ = stab[max(max(dxs[c + 2], dy), dz)], exm = stab[max(max(dxs[c], dy), dz)];
      const float eyp = stab[max(max(dx, dyp), dz)], eym = stab[max(max(dx, dym), dz)];
      const float ezp = stab[max(dxy, dzp)], ezm = stab[max(dxy, dzm)];
      const float g = __fadd_rn(__fadd_rn(gterm(exp_, exm, f4get(xp, c), f4get(xm, c), G.i2hx),
                                          gterm(eyp, eym, f4get(yp, c), f4get(ym, c), G.i2hy)),
                                gterm(ezp, ezm, f4get(zp, c), f4get(zm, c), G.i2hz));
      res[c] = upd_pml(Lc, g, uc, upc, vc, stab[G.T + d], stab[2 * G.T + d]);
    }
  }
  return make_float4(res[0], res[1], res[2], res[3]);
}

template <int TX, int CW, int TY, int TYT, int MODE, int MINB, int RA = 0>
__global__ void __maxnreg__((StreamCfg<TX, CW, TY, TYT, MINB, RA>::MAXR))
k_stream(const __grid_constant__ CUtensorMap tm_u,    // u^n, box (TX+8, TY+8, 1)
         const __grid_constant__ CUtensorMap tm_up,   // u^{n-1}, box (CW, TY, 1)
         const __grid_constant__ CUtensorMap tm_v,    // vdt2, box (CW, TY, 1)
         const __grid_constant__ StreamParams P) {
  using C = StreamCfg<TX, CW, TY, TYT, MINB, RA>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* su = reinterpret_cast<float*>(smem_raw);
  float* sup = su + SU * C::U_STAGE;
  float* sv = sup + SP * C::P_STAGE;
  uint64_t* full_u = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
  uint64_t* empty_u = full_u + SU;
  uint64_t* full_p = empty_u + SU;
  uint64_t* empty_p = full_p + SP;
  float* stab = reinterpret_cast<float*>(smem_raw + C::TAB_OFF);
  const int TABN = P.w + 2;

  // ---- work unit ---------------------------------------------------------
  int b = blockIdx.x, ri = 0;
#pragma unroll 1
  while (ri + 1 < P.nreg && b >= P.reg[ri + 1].blk0) ++ri;
  const Region& G = P.reg[ri];
  b -= G.blk0;
  const int ncol = G.ntx * G.nty;
  const int zc = b / ncol;
  const int rem = b - zc * ncol;
  int tyi, txi;
  if (P.order <= 0) {
    tyi = rem / G.ntx;
    txi = rem - tyi * G.ntx;
  } else {                                 // groups of P.order x-tiles; inside a group y-major
    const int grp = rem / (P.order * G.nty);
    const int gsz = min(P.order, G.ntx - grp * P.order);
    const int r2 = rem - grp * P.order * G.nty;
    tyi = r2 / gsz;
    txi = grp * P.order + (r2 - tyi * gsz);
  }
  const int cx0 = G.ax0 + txi * CW;                       // first computed column
  const int cxo = min(((cx0 % TX) + TX) % TX, TX - CW);   // its offset inside the TX-wide box
  const int bx0 = cx0 - cxo;                              // box origin (128-B aligned when possible)
  const int ty0 = G.y0 + tyi * TY;
  const int zs = G.z0 + zc * P.cz;
  const int ze = min(zs + P.cz, G.z1);

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;

  // ---- setup: barriers, PML tables --------------------------------------
  if (tid == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_up);
    prefetch_tmap(&tm_v);
#pragma unroll
    for (int s = 0; s < SU; ++s) { mbar_init(&full_u[s], 1); mbar_init(&empty_u[s], C::NWC); }
#pragma unroll
    for (int s = 0; s < SP; ++s) { mbar_init(&full_p[s], 1); mbar_init(&empty_p[s], C::NWC); }
    fence_mbar_init();
  }
  for (int i = tid; i < 3 * TABN; i += C::NT) stab[i] = P.tab[i];
  __syncthreads();

  // ======================= producer warp =================================
  if (wid >= C::NWC) {
    if (RA > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
    if (wid != C::NWC || lane != 0) return;
    const uint64_t pol_u = P.upol ? policy_evict_normal() : policy_evict_last();  // u^n: halo re-reads
    const uint64_t pol_s = policy_evict_first();   // u^{n-1}, vdt2: streamed once
    // u plane p (local z, p >= zs-4) lives in u stage (p - zs + 4) % 9, use (p - zs + 4) / 9
    auto issue_u = [&](int p, int st) {
      mbar_arrive_expect_tx(&full_u[st], C::U_STAGE * 4);
      tma_load_3d(su + st * C::U_STAGE, &tm_u, &full_u[st], bx0 - R, ty0 - R, p + R, pol_u);
    };
    // p plane p (p >= zs) lives in p stage (p - zs) % 3, use (p - zs) / 3
    auto issue_p = [&](int p, int st) {
      mbar_arrive_expect_tx(&full_p[st], 2 * C::P_STAGE * 4);
      tma_load_3d(sup + st * C::P_STAGE, &tm_up, &full_p[st], cx0, ty0, p + R, pol_s);
      tma_load_3d(sv + st * C::P_STAGE, &tm_v, &full_p[st], cx0, ty0, p, pol_s);
    };
    for (int s = 0; s < SU; ++s)
      if (zs - R + s <= ze + R - 1) issue_u(zs - R + s, s);      // planes zs-4 .. zs+4
    for (int s = 0; s < SP; ++s)
      if (zs + s < ze) issue_p(zs + s, s);                       // planes zs .. zs+2
    // refill in release order: when plane t is released, u plane t+9 and p plane t+3 go in
#pragma unroll 1
    for (int t = zs - R; t + SU <= ze + R - 1 || t + SP < ze; ++t) {
      if (t + SU <= ze + R - 1) {
        const int o = t - zs + R;
        mbar_wait(&empty_u[o % SU], (o / SU) & 1);
        issue_u(t + SU, o % SU);
      }
      if (t >= zs && t + SP < ze) {
        const int o = t - zs;
        mbar_wait(&empty_p[o % SP], (o / SP) & 1);
        issue_p(t + SP, o % SP);
      }
      if (P.pf > 0) {
        const int pu = t + SU + P.pf, pp = t + SP + P.pf;
        if (pu <= ze + R - 1) tma_prefetch_3d(&tm_u, bx0 - R, ty0 - R, pu + R);
        if (t >= zs && pp < ze) {
          tma_prefetch_3d(&tm_up, cx0, ty0, pp + R);
          tma_prefetch_3d(&tm_v, cx0, ty0, pp);
        }
      }
    }
    return;
  }

  // ======================= consumer warps ================================
  if (RA > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(RA) : "memory");
  const int lx = (wid % C::WX) * C::LXW + (lane % C::LXW);
  const int ly = (wid / C::WX) * C::LYW + (lane / C::LXW);
  const int gx = cx0 + 4 * lx;              // first x of my float4
  const int gy = ty0 + ly * TYT;            // first y of my rows
  // smem offsets (floats) of my float4 in row 0 of the tile, u stage / p stage
  const int uo = (ly * TYT + R) * C::SW + cxo + 4 * lx + R;
  const int po = (ly * TYT) * CW + 4 * lx;

  // ---- per-thread geometry: store mask, PML coefficients -----------------
  unsigned mask = 0;                         // bit (r*4 + c): point is in the region
#pragma unroll
  for (int r = 0; r < TYT; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int x = gx + c, y = gy + r;
      if (x >= G.x0 && x < G.x1 && y >= G.y0 && y < G.y1) mask |= 1u << (r * 4 + c);
    }
  if (4 * lx >= CW) mask = 0;                // phantom lane beyond the computed width
  const bool full = mask == (TYT * 4 == 32 ? 0xffffffffu : ((1u << (TYT * 4)) - 1u));
  PmlGeo PG;
  PG.nx = P.nx; PG.ny = P.ny; PG.nzg = P.nzg; PG.w = P.w; PG.T = TABN;
  PG.i2hx = P.k.i2h[0]; PG.i2hy = P.k.i2h[1]; PG.i2hz = P.k.i2h[2];
  // fused mode: does any in-region point of my warp lie in the x/y PML?
  bool warp_xy_pml = false;
  if (MODE == MODE_FUSED) {
    bool mine = false;
#pragma unroll
    for (int r = 0; r < TYT; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if ((mask >> (r * 4 + c)) & 1u)
          mine |= dist1(gx + c, P.nx, P.w) > 0 || dist1(gy + r, P.ny, P.w) > 0;
    warp_xy_pml = __any_sync(0xffffffffu, mine);
  }
  // wall mode, planes with dz(k-1) = dz(k) = dz(k+1) = 0: a warp whose points
  // all have dx = 0 (y wall away from the corners) has a row-uniform eta star
  // (grad eta = d_y eta only); one whose points all have dy = 0 (x wall) a
  // column-constant one (d_x eta only).  Precompute those coefficients once:
  //   cg = (eta(+e_a) - eta(-e_a)) / (2 h_a), A_d, B_d
  // Warps mixing both (corners) take the general path.
  int wkind = 0;                             // 1: y-wall rows, 2: x-wall columns, 0: general
  float cgr[TYT], Ar[TYT], Br[TYT];          // y-wall: per row
  float cgc[4], Ac[4], Bc[4];                // x-wall: per column
  if (MODE == MODE_WALL) {
    bool all_dx0 = true, all_dy0 = true;
#pragma unroll
    for (int r = 0; r < TYT; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if ((mask >> (r * 4 + c)) & 1u) {
          all_dx0 &= dist1(gx + c, P.nx, P.w) == 0;
          all_dy0 &= dist1(gy + r, P.ny, P.w) == 0;
        }
    all_dx0 = __all_sync(0xffffffffu, all_dx0);
    all_dy0 = __all_sync(0xffffffffu, all_dy0);
    wkind = all_dx0 ? 1 : (all_dy0 ? 2 : 0);
    // an inner point (d = 0) inside a wall region (the frames of a two-step
    // pair reach 4 or 8 cells into the inner box) takes cg = 0, A = B = 1:
    // ((2u - up) + v (L + 0)) / 1, bitwise the inner update (up to the sign of 0)
#pragma unroll
    for (int r = 0; r < TYT; ++r) {
      const int dy = dist1(gy + r, P.ny, P.w);
      cgr[r] = dy == 0 ? 0.f
                       : __fmul_rn(__fsub_rn(stab[dist1(gy + r + 1, P.ny, P.w)], stab[dist1(gy + r - 1, P.ny, P.w)]),
                                   PG.i2hy);
      Ar[r] = stab[TABN + dy];
      Br[r] = stab[2 * TABN + dy];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int dx = dist1(gx + c, P.nx, P.w);
      cgc[c] = dx == 0 ? 0.f
                       : __fmul_rn(__fsub_rn(stab[dist1(gx + c + 1, P.nx, P.w)], stab[dist1(gx + c - 1, P.nx, P.w)]),
                                   PG.i2hx);
      Ac[c] = stab[TABN + dx];
      Bc[c] = stab[2 * TABN + dx];
    }
  }
  float* optr = P.out + (int64_t)(zs + R) * P.plane + (int64_t)gy * P.pitch + gx;

  // ---- warm-up: planes zs-4 .. zs+3 (stages 0..7, first use) -> queue ----
  float4 q[9][TYT];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    mbar_wait(&full_u[s], 0);
#pragma unroll
    for (int r = 0; r < TYT; ++r) q[s][r] = lds4(su + s * C::U_STAGE + uo + r * C::SW);
  }
  __syncwarp();
  if (lane == 0) {                           // planes zs-4..zs-1 are not needed again
#pragma unroll
    for (int s = 0; s < R; ++s) mbar_arrive(&empty_u[s]);
  }

  const Coef& K = P.k;
  // ---- main loop over planes, unrolled 9x (fixed slots / stages) ---------
#pragma unroll 1
  for (int z0 = zs, j = 0; z0 < ze; z0 += 9, ++j) {
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int z = z0 + s;
      if (z >= ze) break;
      const int sl = (s + 8) % 9;            // slot/stage of the leading plane z+4
      const int sc = (s + 4) % 9;            // slot/stage of plane z
      // 1. leading plane z+4 -> queue
      mbar_wait(&full_u[sl], (j + (s >= 1 ? 1 : 0)) & 1);
#pragma unroll
      for (int r = 0; r < TYT; ++r) q[sl][r] = lds4(su + sl * C::U_STAGE + uo + r * C::SW);

      // 2. Laplacian of all 4*TYT points (interleaved chains)
      const float* S = su + sc * C::U_STAGE + uo;
      float4 Y[TYT + 2 * R];                 // rows -4 .. TYT+3 at my float4
#pragma unroll
      for (int jj = 0; jj < TYT + 2 * R; ++jj) {
        if (jj >= R && jj < R + TYT) Y[jj] = q[sc][jj - R];
        else Y[jj] = lds4(S + (jj - R) * C::SW);
      }
      float4 Lf[TYT], Rf[TYT];
#pragma unroll
      for (int r = 0; r < TYT; ++r) {
        Lf[r] = lds4(S + r * C::SW - 4);
        Rf[r] = lds4(S + r * C::SW + 4);
      }
      float L[TYT][4];
#pragma unroll
      for (int r = 0; r < TYT; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) L[r][c] = __fmul_rn(K.c0, f4get(Y[R + r], c));
      if (MODE != MODE_NULL) {
#pragma unroll
      for (int m = 1; m <= R; ++m)
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          const float X[12] = {Lf[r].x, Lf[r].y, Lf[r].z, Lf[r].w, Y[R + r].x, Y[R + r].y,
                               Y[R + r].z, Y[R + r].w, Rf[r].x, Rf[r].y, Rf[r].z, Rf[r].w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
            L[r][c] = __fmaf_rn(K.cx[m - 1], __fadd_rn(X[4 + c + m], X[4 + c - m]), L[r][c]);
        }
#pragma unroll
      for (int m = 1; m <= R; ++m)
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            L[r][c] = __fmaf_rn(K.cy[m - 1], __fadd_rn(f4get(Y[R + r + m], c), f4get(Y[R + r - m], c)), L[r][c]);
#pragma unroll
      for (int m = 1; m <= R; ++m)
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            L[r][c] = __fmaf_rn(K.cz[m - 1],
                                __fadd_rn(f4get(q[(s + 4 + m) % 9][r], c), f4get(q[(s + 4 - m + 9) % 9][r], c)),
                                L[r][c]);
      }

      // 3. u^{n-1}, vdt2 of plane z
      const int sp = s % 3;
      mbar_wait(&full_p[sp], (j + s / 3) & 1);
      float4 upv[TYT], vv[TYT];
#pragma unroll
      for (int r = 0; r < TYT; ++r) {
        upv[r] = lds4(sup + sp * C::P_STAGE + po + r * CW);
        vv[r] = lds4(sv + sp * C::P_STAGE + po + r * CW);
      }
      // all smem reads of plane z done: release its stages to the producer
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_u[sc]);
        mbar_arrive(&empty_p[sp]);
      }

      // 4. update (one uniform branch per plane) and store
      const int kg = z + P.zoff;
      float4 res[TYT];
      if (MODE == MODE_NULL) {
#pragma unroll
        for (int r = 0; r < TYT; ++r)
          res[r] = make_float4(upv[r].x + vv[r].x + L[r][0], upv[r].y + vv[r].y, upv[r].z + vv[r].z,
                               upv[r].w + vv[r].w);
      } else if (MODE == MODE_INNER || (MODE == MODE_FUSED && !warp_xy_pml)) {
        if (kg >= P.w && kg < P.nzg - P.w) {
#pragma unroll
          for (int r = 0; r < TYT; ++r) {
            const float4 Cu = Y[R + r];
            res[r] = make_float4(upd_inner(L[r][0], Cu.x, upv[r].x, vv[r].x),
                                 upd_inner(L[r][1], Cu.y, upv[r].y, vv[r].y),
                                 upd_inner(L[r][2], Cu.z, upv[r].z, vv[r].z),
                                 upd_inner(L[r][3], Cu.w, upv[r].w, vv[r].w));
          }
        } else {
          const int dz = dist1(kg, P.nzg, P.w);
          CapC cc;
          cc.ex = stab[dz];
          cc.ezp = stab[dist1(kg + 1, P.nzg, P.w)];
          cc.ezm = stab[dist1(kg - 1, P.nzg, P.w)];
          cc.A = stab[TABN + dz];
          cc.B = stab[2 * TABN + dz];
#pragma unroll
          for (int r = 0; r < TYT; ++r) {
            const float4 Cu = Y[R + r];
            const float4 xp = make_float4(Cu.y, Cu.z, Cu.w, Rf[r].x);
            const float4 xm = make_float4(Lf[r].w, Cu.x, Cu.y, Cu.z);
            res[r] = cap_update(make_float4(L[r][0], L[r][1], L[r][2], L[r][3]), Cu, upv[r], vv[r], xp, xm,
                                Y[R + r + 1], Y[R + r - 1], q[(s + 5) % 9][r], q[(s + 3) % 9][r], cc,
                                K.i2h[0], K.i2h[1], K.i2h[2]);
          }
        }
      } else if (MODE == MODE_WALL && wkind != 0 && kg > P.w && kg < P.nzg - P.w - 1) {
        // wall, z-interior plane, pure y-wall rows (g = gy) or pure x-wall
        // columns (g = gx); the other two grad terms are +-0 exactly (dropped)
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          const float4 Cu = Y[R + r];
          const float X[12] = {Lf[r].x, Lf[r].y, Lf[r].z, Lf[r].w, Cu.x, Cu.y,
                               Cu.z, Cu.w, Rf[r].x, Rf[r].y, Rf[r].z, Rf[r].w};
          float o[4];
          if (wkind == 1) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float gya = __fmul_rn(cgr[r], __fmul_rn(__fsub_rn(f4get(Y[R + r + 1], c),
                                                                      f4get(Y[R + r - 1], c)), K.i2h[1]));
              o[c] = upd_pml(L[r][c], gya, X[4 + c], f4get(upv[r], c), f4get(vv[r], c), Ar[r], Br[r]);
            }
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float gxa = __fmul_rn(cgc[c], __fmul_rn(__fsub_rn(X[5 + c], X[3 + c]), K.i2h[0]));
              o[c] = upd_pml(L[r][c], gxa, X[4 + c], f4get(upv[r], c), f4get(vv[r], c), Ac[c], Bc[c]);
            }
          }
          res[r] = make_float4(o[0], o[1], o[2], o[3]);
        }
      } else {
        // wall plane in / next to a z cap, or a fused-mode warp touching the x/y
        // PML: full 7-point eta star per point (d = 0 points take the inner formula)
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          const float4 Cu = Y[R + r];
          const float4 xp = make_float4(Cu.y, Cu.z, Cu.w, Rf[r].x);
          const float4 xm = make_float4(Lf[r].w, Cu.x, Cu.y, Cu.z);
          res[r] = pml_row_call(make_float4(L[r][0], L[r][1], L[r][2], L[r][3]), Cu, upv[r], vv[r], xp, xm,
                                Y[R + r + 1], Y[R + r - 1], q[(s + 5) % 9][r], q[(s + 3) % 9][r], gx, gy + r,
                                kg, PG, stab);
        }
      }
      if (full) {
#pragma unroll
        for (int r = 0; r < TYT; ++r) st_cs_f4(optr + r * P.pitch, res[r]);
      } else {
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (mask & (1u << (r * 4 + c))) optr[r * P.pitch + c] = f4get(res[r], c);
      }
      // fused halo exchange: edge planes also go straight into the neighbour's
      // ghost planes over the peer mapping (plane-uniform branch)
      float* rbase = nullptr;
      if (z < R && P.rlo) rbase = P.rlo + (int64_t)z * P.plane;
      else if (z >= P.nzl - R && P.rhi) rbase = P.rhi + (int64_t)(z - (P.nzl - R)) * P.plane;
      if (rbase) {
        float* rp = rbase + (int64_t)gy * P.pitch + gx;
        if (full) {
#pragma unroll
          for (int r = 0; r < TYT; ++r) *reinterpret_cast<float4*>(rp + r * P.pitch) = res[r];
        } else {
#pragma unroll
          for (int r = 0; r < TYT; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (mask & (1u << (r * 4 + c))) rp[r * P.pitch + c] = f4get(res[r], c);
        }
      }
      optr += P.plane;
    }
  }
}

}  // namespace w25
