// tb2.cuh -- two-step temporal blocking ("3.5D") of the z-streaming stencil
// for sm_100a: SURVEY.md §8(f) rank 1, the paper's stated future work
// (PAPER.md L146-157, L1491-1492).  One launch advances the inner column
// from (u^n, u^{n-1}) to (u^{n+1}, u^{n+2}) while reading u^n, u^{n-1} and
// vdt2 from HBM once and writing both new planes once: 20 B per point per
// TWO steps (10 B/point-step) instead of 2 x 16 B.
//
// Work unit: an output tile of TX x TY points (step-2 region S2) x one
// z-chunk [zs, ze).  Step 1 computes u^{n+1} on S1 = S2 grown by the stencil
// radius 4 in x and y (the halo ring is recomputed redundantly, never
// exchanged) and on planes [zs-4, ze+4); step 2 computes u^{n+2} on S2, 4
// planes behind step 1.  Buffers are out of place: (A = u^n, B = u^{n-1}) ->
// (C = u^{n+1}, D = u^{n+2}); neighbouring tiles read A and B while C and D
// are written, so tiles are independent.
//
//  * producer warp: TMA (cp.async.bulk.tensor.3d) of u^n boxes
//    (TX+16) x (TY+16) into a 9-stage ring, of u^{n-1}/vdt2 boxes over S1
//    into a 3-stage ring, of vdt2 over S2 (for step 2; an L2 hit, the plane
//    was fetched 4 planes earlier) into a 3-stage ring; full/empty mbarriers.
//  * consumer thread = one float4 of S1 row r1 (16 lanes x 2 rows per warp
//    for TX = 56).  Step 1: x/y neighbours from the u^n ring, z neighbours from
//    a 9-slot register queue q1 (the paper's st_reg_fixed).
//    u^{n+1} goes to global C (own S2 points), to a shared ring U1 (for the
//    x/y neighbours of step 2; full/empty mbarriers between warps) and to a
//    second 9-slot register queue q2 (z neighbours of step 2).  Step 2 runs
//    in the warps whose rows lie in S2 (warp-uniform) with u^{n-1} := u^n
//    taken from q1 (the oldest slot).
//  * per-point arithmetic identical to k_stream / k_naive (common.cuh):
//    the result is bitwise equal to two single steps.
//  * the source is injected where it is computed: step 1 (including the
//    redundant halo copies) adds inc[n], step 2 adds inc[n+1]; n = *dstep.
//  * MODE_INNER only: S1 must lie in the inner xy box; z caps are
//    plane-uniform (cap_update); planes outside [0, nz) are the zero fringe.
#pragma once
#include "stream.cuh"

namespace w25 {

struct T2Params {
  float* outC;                  // u^{n+1} buffer (padded layout base)
  float* outD;                  // u^{n+2} buffer
  int64_t pitch, plane;
  int nx, ny, nzl, nzg, zoff, w;
  int cz;                       // z-chunk length
  int ax0, ay0;                 // tile grid origin (S2 top-left of tile 0, ax0 % 4 == 0)
  int ntx, nty, nzc;            // tiles in x, y and z-chunks
  int dx0, dx1, dy0, dy1;       // D (u^{n+2}) store box
  int cx0, cx1, cy0, cy1;       // C (u^{n+1}) store box
  Coef k;
  const float* tab;             // [3][w+2]
  // source (local z plane sk < 0: none on this plan)
  int si, sj, sk;
  const float* inc;
  int64_t ninc;
  const unsigned long long* dstep;
};

template <int TX, int TY>
struct T2Cfg {
  static constexpr int W1 = TX + 2 * R, H1 = TY + 2 * R;      // S1
  static constexpr int W0 = TX + 4 * R, H0 = TY + 4 * R;      // u^n box
  static constexpr int LX = W1 / 4;                           // float4 lanes per row
  static constexpr int LY = 32 / LX;                          // rows per warp
  static constexpr int NWC = H1 / LY;                         // consumer warps
  static constexpr int NT = 32 * (NWC + 1);
  static constexpr int W2A = R / LY, W2B = (TY + R) / LY;     // step-2 warps [W2A, W2B)
  static constexpr int NW2 = W2B - W2A;
  // register cap: warps are spread round-robin over the 4 sub-partitions, each
  // with a 16K-register file
  static constexpr int WPS = (NWC + 1 + 3) / 4;
  static constexpr int MAXR_ = (16384 / (32 * WPS)) & ~7;
  static constexpr int MAXR = MAXR_ > 255 ? 255 : MAXR_;
  static constexpr int NU1 = 6;                               // u^{n+1} shared ring slots
  static constexpr int S0F = W0 * H0, S1F = W1 * H1, S2F = TX * TY;   // floats per box
  static constexpr int rnd(int n) { return (n + 31) / 32 * 32; }       // 128-B stage strides
  static constexpr int S0S = rnd(S0F), S1S = rnd(S1F), S2S = rnd(S2F);
  static constexpr int OFF_UP = SU * S0S;                     // float offsets
  static constexpr int OFF_V1 = OFF_UP + SP * S1S;
  static constexpr int OFF_V2 = OFF_V1 + SP * S1S;
  static constexpr int OFF_U1 = OFF_V2 + SP * S2S;
  static constexpr int BAR_OFF = (OFF_U1 + NU1 * S1S) * 4;    // bytes
  static constexpr int NBAR = 2 * SU + 2 * SP + 2 * SP + 2 * NU1;
  static constexpr int TAB_OFF = BAR_OFF + NBAR * 8;
  static size_t smem_bytes(int w) { return TAB_OFF + 3 * (w + 2) * 4; }
  static_assert(32 % LX == 0 && LX >= 4, "S1 width must be 16, 32, 64 or 128 floats");
  static_assert(R % LY == 0 && TY % LY == 0, "step-2 rows must be whole warps");
  static_assert(TX % 4 == 0, "tile width");
};

// Laplacian of one float4 (4 x-consecutive points), Eq. 3:
// c_xyz u, then pair sums along x, y, z for m = 1..4 (same order as lap8).
__device__ __forceinline__ void lap_f4(const Coef& K, float L[4], float4 C, float4 Lf, float4 Rf,
                                       const float4 (&Ym)[R], const float4 (&Yp)[R], const float4 (&Zm)[R],
                                       const float4 (&Zp)[R]) {
  const float X[12] = {Lf.x, Lf.y, Lf.z, Lf.w, C.x, C.y, C.z, C.w, Rf.x, Rf.y, Rf.z, Rf.w};
#pragma unroll
  for (int c = 0; c < 4; ++c) L[c] = __fmul_rn(K.c0, X[4 + c]);
#pragma unroll
  for (int m = 1; m <= R; ++m)
#pragma unroll
    for (int c = 0; c < 4; ++c) L[c] = __fmaf_rn(K.cx[m - 1], __fadd_rn(X[4 + c + m], X[4 + c - m]), L[c]);
#pragma unroll
  for (int m = 1; m <= R; ++m)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      L[c] = __fmaf_rn(K.cy[m - 1], __fadd_rn(f4get(Yp[m - 1], c), f4get(Ym[m - 1], c)), L[c]);
#pragma unroll
  for (int m = 1; m <= R; ++m)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      L[c] = __fmaf_rn(K.cz[m - 1], __fadd_rn(f4get(Zp[m - 1], c), f4get(Zm[m - 1], c)), L[c]);
}

// Update of one float4 at global plane kg: inner formula, or the plane-uniform
// z-cap PML update (x, y inner), or the zero fringe outside [0, nzg).
__device__ __forceinline__ float4 upd_col(const T2Params& P, const float* stab, int kg, const float L[4],
                                          float4 C, float4 up, float4 v, float4 Lf, float4 Rf, float4 ym1,
                                          float4 yp1, float4 zm1, float4 zp1) {
  if (kg >= P.w && kg < P.nzg - P.w) {
    return make_float4(upd_inner(L[0], C.x, up.x, v.x), upd_inner(L[1], C.y, up.y, v.y),
                       upd_inner(L[2], C.z, up.z, v.z), upd_inner(L[3], C.w, up.w, v.w));
  }
  if (kg < 0 || kg >= P.nzg) return make_float4(0.f, 0.f, 0.f, 0.f);
  const int T = P.w + 2;
  const int dz = dist1(kg, P.nzg, P.w);
  CapCT<float> cc;
  cc.ex = stab[dz];
  cc.ezp = stab[dist1(kg + 1, P.nzg, P.w)];
  cc.ezm = stab[dist1(kg - 1, P.nzg, P.w)];
  cc.A = stab[T + dz];
  cc.B = stab[2 * T + dz];
  const float4 xp = make_float4(C.y, C.z, C.w, Rf.x);
  const float4 xm = make_float4(Lf.w, C.x, C.y, C.z);
  return cap_update<float>(make_float4(L[0], L[1], L[2], L[3]), C, up, v, xp, xm, yp1, ym1, zp1, zm1, cc, P.k.i2h[0],
                    P.k.i2h[1], P.k.i2h[2]);
}

__device__ __forceinline__ float4 f4add_at(float4 a, int c, float v) {
  if (c == 0) a.x = __fadd_rn(a.x, v);
  else if (c == 1) a.y = __fadd_rn(a.y, v);
  else if (c == 2) a.z = __fadd_rn(a.z, v);
  else a.w = __fadd_rn(a.w, v);
  return a;
}

template <int TX, int TY>
__global__ void __maxnreg__((T2Cfg<TX, TY>::MAXR))
k_tb2(const __grid_constant__ CUtensorMap tm_u,    // A = u^n, box (W0, H0, 1)
      const __grid_constant__ CUtensorMap tm_up,   // B = u^{n-1}, box (W1, H1, 1)
      const __grid_constant__ CUtensorMap tm_v1,   // vdt2, box (W1, H1, 1)
      const __grid_constant__ CUtensorMap tm_v2,   // vdt2, box (TX, TY, 1)
      const __grid_constant__ T2Params P) {
  using C = T2Cfg<TX, TY>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sf = reinterpret_cast<float*>(smem_raw);
  float* su = sf;
  float* sup = sf + C::OFF_UP;
  float* sv1 = sf + C::OFF_V1;
  float* sv2 = sf + C::OFF_V2;
  float* su1 = sf + C::OFF_U1;
  uint64_t* full_u = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
  uint64_t* empty_u = full_u + SU;
  uint64_t* full_p = empty_u + SU;
  uint64_t* empty_p = full_p + SP;
  uint64_t* full_v = empty_p + SP;
  uint64_t* empty_v = full_v + SP;
  uint64_t* full_1 = empty_v + SP;
  uint64_t* empty_1 = full_1 + C::NU1;
  float* stab = reinterpret_cast<float*>(smem_raw + C::TAB_OFF);   // PML tables (z caps)

  // ---- work unit (chunk-major, x fastest) --------------------------------
  const int b = blockIdx.x;
  const int ncol = P.ntx * P.nty;
  const int zc = b / ncol;
  const int rem = b - zc * ncol;
  const int tyi = rem / P.ntx, txi = rem - tyi * P.ntx;
  const int x0 = P.ax0 + txi * TX, y0 = P.ay0 + tyi * TY;
  const int zs = zc * P.cz;
  const int ze = min(zs + P.cz, P.nzl);
  const int nit = ze - zs + 2 * R;          // iterations: step-1 planes zs-4 .. ze+3

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_up);
    prefetch_tmap(&tm_v1);
    prefetch_tmap(&tm_v2);
#pragma unroll
    for (int s = 0; s < SU; ++s) { mbar_init(&full_u[s], 1); mbar_init(&empty_u[s], C::NWC); }
#pragma unroll
    for (int s = 0; s < SP; ++s) {
      mbar_init(&full_p[s], 1); mbar_init(&empty_p[s], C::NWC);
      mbar_init(&full_v[s], 1); mbar_init(&empty_v[s], C::NW2);
    }
#pragma unroll
    // U1 (thread-written, read by other warps): every writer thread arrives
    // (release of its own store), so the reader's acquire covers each store
    for (int s = 0; s < C::NU1; ++s) { mbar_init(&full_1[s], C::NWC * 32); mbar_init(&empty_1[s], C::NW2 * 32); }
    fence_mbar_init();
  }
  const int TABN = P.w + 2;
  for (int i = tid; i < 3 * TABN; i += C::NT) stab[i] = P.tab[i];
  __syncthreads();

  // ======================= producer warp =================================
  if (wid == C::NWC) {
    if (lane != 0) return;
    const uint64_t pol_u = policy_evict_last();    // u^n: halo re-reads by neighbour tiles
    const uint64_t pol_n = policy_evict_normal();  // u^{n-1}, vdt2 (S1): halos + the S2 re-read
    const uint64_t pol_f = policy_evict_first();   // vdt2 (S2) for step 2: last use
    const int zu0 = zs - 2 * R;                    // first u^n plane
    const int zu1 = ze + 2 * R - 1;                // last u^n plane
    auto issue_u = [&](int p, int st) {
      mbar_arrive_expect_tx(&full_u[st], C::S0F * 4);
      tma_load_3d(su + st * C::S0S, &tm_u, &full_u[st], x0 - 2 * R, y0 - 2 * R, p + R, pol_u);
    };
    auto issue_p = [&](int z, int st) {            // step-1 plane z
      mbar_arrive_expect_tx(&full_p[st], 2 * C::S1F * 4);
      tma_load_3d(sup + st * C::S1S, &tm_up, &full_p[st], x0 - R, y0 - R, z + R, pol_n);
      tma_load_3d(sv1 + st * C::S1S, &tm_v1, &full_p[st], x0 - R, y0 - R, z, pol_n);
    };
    auto issue_v = [&](int z, int st) {            // step-2 plane z
      mbar_arrive_expect_tx(&full_v[st], C::S2F * 4);
      tma_load_3d(sv2 + st * C::S2S, &tm_v2, &full_v[st], x0, y0, z, pol_f);
    };
    for (int s = 0; s < SU; ++s) issue_u(zu0 + s, s);                       // zs-8 .. zs
    for (int s = 0; s < SP; ++s) issue_p(zs - R + s, s);                   // zs-4 .. zs-2
    for (int s = 0; s < SP; ++s)
      if (zs + s < ze) issue_v(zs + s, s);                                  // zs .. zs+2
    // refill in release order; all three releases of index t happen in the
    // consumers' iteration z1 = t (u^n centre t, step-1 plane t, step-2 plane t-4)
#pragma unroll 1
    for (int t = zu0; t <= ze; ++t) {
      if (t + SU <= zu1) {                       // u plane t released -> plane t+9
        const int o = t - zu0;
        mbar_wait(&empty_u[o % SU], (o / SU) & 1);
        fence_proxy_async_smem();               // generic reads before the async-proxy overwrite
        issue_u(t + SU, o % SU);
      }
      if (t >= zs - R && t + SP <= ze + R - 1) {  // step-1 plane t released -> t+3
        const int o = t - (zs - R);
        mbar_wait(&empty_p[o % SP], (o / SP) & 1);
        fence_proxy_async_smem();
        issue_p(t + SP, o % SP);
      }
      const int tv = t - R;                      // step-2 plane tv released -> tv+3
      if (tv >= zs && tv + SP < ze) {
        const int o = tv - zs;
        mbar_wait(&empty_v[o % SP], (o / SP) & 1);
        fence_proxy_async_smem();
        issue_v(tv + SP, o % SP);
      }
    }
    return;
  }

  // ======================= consumer warps ================================
  const int c4 = lane % C::LX;                    // float4 column in S1
  const int r1 = wid * C::LY + lane / C::LX;      // row in S1
  const bool w2 = wid >= C::W2A && wid < C::W2B;  // warp computes step 2 (uniform)
  const int gx = x0 - R + 4 * c4;                 // global x of my float4
  const int gy = y0 - R + r1;
  const int uo = (r1 + R) * C::W0 + 4 * c4 + R;   // my float4 in a u^n stage
  const int po = r1 * C::W1 + 4 * c4;             // ... in an S1 stage (u^{n-1}, vdt2, U1)
  const int c2 = min(max(c4 - 1, 0), TX / 4 - 1);
  const int vo = max(r1 - R, 0) * TX + 4 * c2;    // ... in an S2 stage (clamped for halo lanes)
  const bool in_s2 = c4 >= 1 && c4 < C::LX - 1 && r1 >= R && r1 < TY + R;
  unsigned mC = 0, mD = 0;                        // per-component store masks
  if (in_s2) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int x = gx + c;
      if (x >= P.cx0 && x < P.cx1 && gy >= P.cy0 && gy < P.cy1) mC |= 1u << c;
      if (x >= P.dx0 && x < P.dx1 && gy >= P.dy0 && gy < P.dy1) mD |= 1u << c;
    }
  }
  // source: component of my float4 holding (si, sj), or -1
  const int src_c = (P.sk >= 0 && gy == P.sj && P.si >= gx && P.si < gx + 4) ? P.si - gx : -1;
  float* pC = P.outC + (int64_t)gy * P.pitch + gx;
  float* pD = P.outD + (int64_t)gy * P.pitch + gx;
  const Coef& K = P.k;

  float4 q1[9], q2[9];
  // ---- warm-up: u^n planes zs-8 .. zs-1 (stages 0..7) -> q1 slots 0..7 ---
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    mbar_wait(&full_u[s], 0);
    q1[s] = lds4(su + s * C::S0S + uo);
  }
  __syncwarp();
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < R; ++s) mbar_arrive(&empty_u[s]);   // planes zs-8..zs-5: never a centre
  }
#pragma unroll
  for (int s = 0; s < 9; ++s) q2[s] = make_float4(0.f, 0.f, 0.f, 0.f);

  int u1w = 0, u1r = 0;                           // U1 ring: planes written / read so far

  // ---- main loop: iteration i = step-1 plane z1 = zs-4+i, unrolled 9x ---
#pragma unroll 1
  for (int i0 = 0, j = 0; i0 < nit; i0 += 9, ++j) {
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i = i0 + s;
      if (i >= nit) break;
      const int z1 = zs - R + i;
      // 1. leading u^n plane z1+4 -> q1 slot (s+8)%9
      const int sl = (s + 8) % 9, sc = (s + 4) % 9;
      mbar_wait(&full_u[sl], (j + (s >= 1 ? 1 : 0)) & 1);
      q1[sl] = lds4(su + sl * C::S0S + uo);
      // 2. step 1 at z1: x/y neighbours from the u^n stage, z from q1
      {
        const float* S = su + sc * C::S0S + uo;
        const float4 Cu = q1[sc];
        const float4 Lf = lds4(S - 4), Rf = lds4(S + 4);
        float4 Ym[R], Yp[R], Zm[R], Zp[R];
#pragma unroll
        for (int m = 1; m <= R; ++m) {
          Ym[m - 1] = lds4(S - m * C::W0);
          Yp[m - 1] = lds4(S + m * C::W0);
          Zm[m - 1] = q1[(s + 4 - m + 9) % 9];
          Zp[m - 1] = q1[(s + 4 + m) % 9];
        }
        float L[4];
        lap_f4(K, L, Cu, Lf, Rf, Ym, Yp, Zm, Zp);
        const int sp = s % 3;
        mbar_wait(&full_p[sp], (j + s / 3) & 1);
        const float4 upv = lds4(sup + sp * C::S1S + po);
        const float4 vv = lds4(sv1 + sp * C::S1S + po);
        __syncwarp();
        if (lane == 0) { mbar_arrive(&empty_u[sc]); mbar_arrive(&empty_p[sp]); }
        const int kg = z1 + P.zoff;
        float4 u1 = upd_col(P, stab, kg, L, Cu, upv, vv, Lf, Rf, Ym[0], Yp[0], Zm[0], Zp[0]);
        if (src_c >= 0 && z1 == P.sk) {
          const unsigned long long n = *P.dstep;
          if (n < (unsigned long long)P.ninc) u1 = f4add_at(u1, src_c, P.inc[n]);
        }
        // 3. u^{n+1}: global C (own S2 points, planes in the chunk), q2, U1
        if (i >= R && i < nit - R) {
          if (mC == 0xfu) st_cs_f4(pC + (int64_t)(z1 + R) * P.plane, u1);
          else if (mC) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (mC & (1u << c)) pC[(int64_t)(z1 + R) * P.plane + c] = f4get(u1, c);
          }
          // U1 write (plane index u1w = i - 4); slot reuse waits for step-2 readers
          const int slot = u1w % C::NU1, use = u1w / C::NU1;
          if (use > 0) mbar_wait(&empty_1[slot], (use - 1) & 1);
          *reinterpret_cast<float4*>(su1 + slot * C::S1S + po) = u1;
          mbar_arrive(&full_1[slot]);
          ++u1w;
        }
        q2[s] = u1;                               // slot i % 9 = s
      }
      // 4. step 2 at z2 = z1 - 4 (warps with S2 rows)
      if (i >= 2 * R && w2) {
        const int z2 = z1 - R;
        const int slot = u1r % C::NU1, use = u1r / C::NU1;
        mbar_wait(&full_1[slot], use & 1);
        const float* S = su1 + slot * C::S1S + po;
        const float4 Cu = q2[(s + 5) % 9];
        const float4 Lf = lds4(S - 4), Rf = lds4(S + 4);
        float4 Ym[R], Yp[R], Zm[R], Zp[R];
#pragma unroll
        for (int m = 1; m <= R; ++m) {
          Ym[m - 1] = lds4(S - m * C::W1);
          Yp[m - 1] = lds4(S + m * C::W1);
          Zm[m - 1] = q2[(s + 5 - m + 9) % 9];
          Zp[m - 1] = q2[(s + 5 + m) % 9];
        }
        float L[4];
        lap_f4(K, L, Cu, Lf, Rf, Ym, Yp, Zm, Zp);
        const int iv = i - 2 * R;                 // step-2 plane index z2 - zs
        const int sv = iv % SP;
        mbar_wait(&full_v[sv], (iv / SP) & 1);
        const float4 vv = lds4(sv2 + sv * C::S2S + vo);
        mbar_arrive(&empty_1[slot]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_v[sv]);
        ++u1r;
        const float4 upv = q1[s % 9];             // u^n(z2): the oldest q1 slot
        const int kg = z2 + P.zoff;
        float4 u2 = upd_col(P, stab, kg, L, Cu, upv, vv, Lf, Rf, Ym[0], Yp[0], Zm[0], Zp[0]);
        if (src_c >= 0 && z2 == P.sk) {
          const unsigned long long n = *P.dstep + 1;
          if (n < (unsigned long long)P.ninc) u2 = f4add_at(u2, src_c, P.inc[n]);
        }
        if (mD == 0xfu) st_cs_f4(pD + (int64_t)(z2 + R) * P.plane, u2);
        else if (mD) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (mD & (1u << c)) pD[(int64_t)(z2 + R) * P.plane + c] = f4get(u2, c);
        }
      } else if (i >= 2 * R && !w2) {
        // keep the U1 read counter in step with the step-2 warps (no reads)
        ++u1r;
      }
    }
  }
}

}  // namespace w25
