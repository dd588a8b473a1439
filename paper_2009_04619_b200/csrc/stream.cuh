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
//  * Precision T = float (production) or double (fp64 plans): every lane holds
//    one 16-byte vector V = float4 / double2, i.e. NV = 4 / 2 x-points.
//  * Each consumer thread owns NV consecutive x points (one V) x TYT rows
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
// MODE_WALL_ETA: wall kernel reading a stored (user-supplied) eta field.
// MODE_WALLX / MODE_WALLY: MODE_WALL specialised for the x walls (only the
// column-constant fast path compiled) / the y walls (row-uniform fast path):
// half the hot-loop code (ncu: instruction-fetch stalls in the generic wall
// kernel); other warps fall back to the general path, so any region is correct.
// MODE_SEAM: the two x walls as "seams" -- seam t = [right wall of row t-1 |
// left wall of row t], 2w contiguous points of one 128-B line (fp32, w = 16,
// rows of exactly nx elements, the layout's origin shift).  The
// region's x range is [R, R + 2w) and y range the seam index t in [0, ny + 1)
// of seam tensor maps whose column 0 is x = nx - w - R of row t - 1.  Only the
// column-constant fast path is compiled (like MODE_WALLX).
// MODE_INNER_EW: MODE_INNER whose producer warpgroup also computes the PML
// walls -- two "wall warps" stream 16 x 8 wall tiles through their own small
// TMA ring while the consumer warps stream the interior tile.
enum { MODE_INNER = 0, MODE_WALL = 1, MODE_NULL = 2, MODE_FUSED = 3, MODE_WALL_ETA = 4, MODE_WALLX = 5,
       MODE_WALLY = 6, MODE_SEAM = 7, MODE_INNER_EW = 8 };

struct Region {
  int x0, x1, y0, y1, z0, z1;   // point box [x0,x1) x [y0,y1) x [z0,z1) (local z)
  int ax0;                      // x0 rounded down to a multiple of 4 (first computed column)
  int ntx, nty, nzc;            // tiles in x (step CW), y (step TY) and z-chunks
  int blk0;                     // first blockIdx.x of this region
};

constexpr int MAX_REGIONS = 4;
constexpr int EW_MAX_REG = 8;   // wall regions of an embedded-wall launch (4 xy boxes x 2 z ranges)
constexpr int SU = 9;           // u ring stages  (= 2R+1)
constexpr int SP = 3;           // u_prev/vdt2 ring stages of the TB2 kernel (divides 9)
#ifndef W25_PACKED
#define W25_PACKED 1            // fp32 Laplacian on packed pairs (FFMA2); -DW25_PACKED=0 for the scalar A/B build
#endif
#ifndef W25_PACK_WALLY
#define W25_PACK_WALLY 0        // y-wall Laplacian on packed pairs too (A/B build: -DW25_PACK_WALLY=1)
#endif
#ifndef W25_PACK_WALLX
#define W25_PACK_WALLX 0        // x-wall Laplacian on packed pairs (A/B build: -DW25_PACK_WALLX=1)
#endif
#ifndef W25_SP_MAX
#define W25_SP_MAX 4            // deepest u_prev/vdt2 ring k_stream may use (A/B builds: -DW25_SP_MAX=3)
#endif
constexpr int W25_MAX_W = 256;  // largest PML width (the shared tables hold 4 (w + 2) entries; 256 leaves the
                                // x walls room for a 4-stage u_prev/vdt2 ring)
constexpr int W25_SMEM_BUDGET = 232448 - 4096;   // 227 KB opt-in limit minus static shared memory

struct StreamParams {
  void* out;                    // u_next buffer (= u_prev buffer), padded layout base (T)
  void* rlo;                    // lower neighbour's upper ghost planes (next buffer) or null
  void* rhi;                    // upper neighbour's lower ghost planes (next buffer) or null
  int64_t pitch, plane;         // row / plane pitch in elements
  int nx, ny, nzl, nzg, zoff, w;
  int cz;                       // z-chunk length
  int pf;                       // L2 prefetch distance (planes beyond the rings; 0 = off)
  int order;                    // tile order in a chunk: 0 = x fastest; G > 0 = groups of G x-tiles, y inside;
                                // -B = bands of B tile rows, y fastest inside a band
  int upol;                     // L2 policy of u loads: 0 = evict_last, 1 = evict_normal
  int nreg;
  Region reg[MAX_REGIONS];
  Coef k;                       // fp32 plans
  CoefT<double> kd;             // fp64 plans
  const void* tab;              // [4][w+2] (T): eta_d, A_d, B_d, RN(1/B_d) (d = 0..w), eta_{w+1} = 0
  int fastdiv;                  // divide by table B values as Markstein n*rB + FMA correction (verified
                                // bitwise == RN(n/B) for this plan's B at setup; common.cuh div_table)
  // tensor maps in global memory (one per buffer, never rewritten) used instead
  // of the __grid_constant__ copies when non-null (WAVE25_GMAPS)
  const CUtensorMap* gu;
  const CUtensorMap* gup;
  const CUtensorMap* gv;
  // stored (user-supplied) eta: [nz][ny][pitch] fp32 or null
  const float* eta;
  double dt;                    // the fp32 dt, widened (A/B = 1 -+ eta dt in fp64)
  // two steps through L2 (PAIR kernels): step-1 blocks read
  // (gu, gup) and write `out`; step-2 blocks read (gu2, gup2) and write `out2`
  // after waiting on the step-1 progress of their own and neighbouring tiles
  const int* pair_groups;       // group g -> role (1, 2) << 16 | tile row
  unsigned* prog;               // per tile: planes completed x consumer warps
  const CUtensorMap* gu2;
  const CUtensorMap* gup2;
  void* out2;
  int src_i, src_j, src_k;      // source cell (local z; src_k < 0: none)
  const void* inc;              // source increments (T)
  int64_t ninc;
  const unsigned long long* dstep;
  int pair_dbg;                 // timing probes only (WAVE25_PAIR_DBG): 1 = no waits, 2 = no publication,
                                // 8 = per-block timeline records
  int pair_pk;                  // step 1 publishes its progress every pair_pk planes (and at the end)
  int64_t pair_dbg_off;         // timeline records (pair_dbg & 8) at prog + this, 6 u64 per block
  int64_t pair_ticket;          // prog[pair_ticket]: next work unit (zeroed with the counters)
  int st_keep;                  // u_next stored with the default (evict-normal) policy instead of
                                // streaming (.cs) stores: the next step re-reads it soon (A/B)
  int inter2;                   // 2 equal regions interleaved block by block (the two x walls: the
                                // right wall of row y and the left wall of row y+1 share a line)
  // stored eta through the u_prev/vdt2 ring (MODE_WALL_ETA): [nz][ny][pitch]
  // fp32, box (CW + 8) x (TY + 2), out-of-range cells (eta = 0) zero-filled
  alignas(64) CUtensorMap tm_eta;
  // embedded walls (MODE_INNER_EW): the PML wall regions, cut into 16 x 8 tiles
  // x z-chunks of cz planes ("units"), claimed by the CTAs' wall warps from a
  // global ticket while their interior tile streams
  struct Ew {
    int nreg;                   // wall regions (same z-chunk count in each)
    Region reg[EW_MAX_REG];     // ntx, nty in 16 x 8 tiles; blk0 = first tile of the region within a chunk
    int cz, ntile, nunits;      // chunk length, tiles per chunk, units (ntile x chunks)
    int min_rem;                // claim while the CTA's interior has >= min_rem planes to go
    int last_blk;               // CTAs >= last_blk (the last wave) also claim once their interior is done
    unsigned* ctr;              // [0] next unit, [1] CTAs whose wall warps have finished (self-resetting)
    int pf;                     // L2 prefetch distance of the wall loads (planes beyond the ring; 0 = off)
    unsigned long long* dbg;    // timing probe (WAVE25_EW_DBG): [0/1] ns, planes claimed during the
                                // interior, [2/3] in the last wave's mop-up, [4/5] units
    alignas(64) CUtensorMap tu; // u^n, box (16 + 2R) x (8 + 2R)
    alignas(64) CUtensorMap tup;  // u^{n-1}, box 16 x 8
    alignas(64) CUtensorMap tv;   // vdt2, box 16 x 8
  } ew;
};

__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acqrel_cta_shared_add(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <typename T> __device__ __forceinline__ const CoefT<T>& coef_of(const StreamParams& P);
template <> __device__ __forceinline__ const CoefT<float>& coef_of<float>(const StreamParams& P) { return P.k; }
template <> __device__ __forceinline__ const CoefT<double>& coef_of<double>(const StreamParams& P) { return P.kd; }

// RA > 0: one CTA per SM with a producer WARPGROUP (4 warps, one issuing TMA)
// that gives its registers back (setmaxnreg.dec to 24) so that the consumer
// warpgroups can raise theirs to RA (setmaxnreg.inc) -- Blackwell/Hopper
// warp-specialised register reallocation.  Needs NWC % 4 == 0.
// embedded wall warps (MODE_INNER_EW): 16 x 8 tiles, two warps of 32 lanes x 2 points
constexpr int EW_CW = 16, EW_TY = 8;
constexpr int EW_SW = EW_CW + 2 * R;                 // u box row (floats)
constexpr int EW_US = EW_SW * (EW_TY + 2 * R);       // u stage (floats)
constexpr int EW_PS = EW_CW * EW_TY;                 // u_prev / vdt2 stage (floats)
constexpr int EW_SPN = 3;                            // u_prev / vdt2 ring depth
constexpr int EW_RP = 64;                            // producer-warpgroup registers (TMA warp + wall warps)
constexpr int EW_RC = 104;                           // consumer registers (512 x 104 + 128 x 64 = 640 x 96)
constexpr int EW_COEF = 64 * 8;                      // per wall lane: cg, A, B, rB of its 2 points (floats)
constexpr int EW_BYTES_ = (SU * EW_US + 2 * EW_SPN * EW_PS + EW_COEF) * 4 + 2 * (SU + EW_SPN) * 8 + 16;
constexpr int EW_BYTES = (EW_BYTES_ + 127) / 128 * 128;

template <int TX, int CW, int TY, int TYT, int MINB = 2, int RA = 0, typename T = float, int ETA = 0, int EWB = 0>
struct StreamCfg {
  static constexpr int NV = VecT<T>::N;                     // x points per lane vector
  static constexpr int LXW = (CW / NV) < 8 ? (CW / NV) : 8; // vector lanes per warp row
  static constexpr int LYW = 32 / LXW;                      // thread rows per warp
  static constexpr int WX = (CW / NV + LXW - 1) / LXW;      // consumer warps across x (the last
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
  // a u box wider than the TMA limit (256) is loaded as NH = 2 half boxes of
  // (TX/2 + 8) x (TY + 8), each with its own halo, side by side in the stage
  static constexpr int NH = (TX + 2 * R > 256) ? 2 : 1;
  static constexpr int HW = TX / NH;                        // half-tile width
  static constexpr int SW = HW + 2 * R;                     // smem u row stride (elements)
  static constexpr int SH = TY + 2 * R;
  static constexpr int U_HALF = SW * SH;
  static constexpr int U_STAGE = NH * U_HALF;               // elements per u stage
  static constexpr int P_STAGE = CW * TY;                   // elements per u_prev / vdt2 stage
  // stored-eta kernels (ETA): an fp32 eta box of (CW + 8) x (TY + 2) per u_prev
  // stage -- the tile with a 1-cell y halo and a 4-cell (16-B) x halo
  // (see SWZ below: 128-B-row u boxes are loaded swizzled and need a 1024-B aligned layout)
  static constexpr bool SWZ_ = NH == 1 && (HW + 2 * R) * (int)sizeof(T) == 128 &&
                               ((HW + 2 * R) * (TY + 2 * R) * (int)sizeof(T)) % 1024 == 0;
  static constexpr int EW = CW + 8;
  static constexpr int E_STAGE = ETA ? (EW * (TY + 2) + 31) / 32 * 32 : 0;  // floats (stages 128-B aligned)
  // u_prev / vdt2 ring depth: as deep as shared memory allows (3..W25_SP_MAX
  // stages), so more of those two streams is in flight per SM
  // (MINB CTAs per SM share its 228 KB, 1 KB reserved per CTA, ~2 KB static)
  static constexpr int BUDGET = MINB > 1 ? (233472 / MINB - 1024 - 2048) : W25_SMEM_BUDGET;
  static constexpr int fits_(int n) {
    return (SWZ_ ? 1024 : 0) + (SU * U_STAGE + 2 * n * P_STAGE) * (int)sizeof(T) + n * E_STAGE * 4 +
               2 * (SU + n) * 8 + (EWB ? EWB + 128 : 0) + 4 * (W25_MAX_W + 2) * (int)sizeof(T) <= BUDGET;
  }
  static constexpr int SPN = (W25_SP_MAX >= 5 && fits_(5)) ? 5 : (W25_SP_MAX >= 4 && fits_(4)) ? 4 : 3;
  static constexpr int E_OFF = (SU * U_STAGE + 2 * SPN * P_STAGE) * (int)sizeof(T);    // bytes (eta ring)
  static constexpr int BAR_OFF = E_OFF + SPN * E_STAGE * 4;                             // bytes
  // embedded wall warps' region (128-B aligned TMA stages), then the PML tables
  static constexpr int EW_OFF = (BAR_OFF + 2 * (SU + SPN) * 8 + 127) / 128 * 128;
  static constexpr int TAB_OFF = EWB ? EW_OFF + EWB : BAR_OFF + 2 * (SU + SPN) * 8;
  // u boxes whose rows are exactly one 128-B line (the fp32 x walls, 24 + 8
  // floats) are loaded with the TMA 128-B swizzle: a float4 column read across
  // the 8 rows of a warp would otherwise hit the same 16 banks (2 wavefronts
  // per 128 B); swizzled stages need 1024-B alignment
  static constexpr bool SWZ = SWZ_;
  static constexpr int ALIGN_PAD = SWZ ? 1024 : 0;
  static size_t smem_bytes(int w) { return ALIGN_PAD + TAB_OFF + 4 * (w + 2) * sizeof(T); }
  static_assert(CW % 4 == 0 && CW <= TX && TX % 4 == 0, "tile widths");
  static_assert(32 % LXW == 0 && (TY / TYT) % LYW == 0 && TY % TYT == 0, "warp tiling");
  static_assert((U_HALF * sizeof(T)) % 128 == 0 && (P_STAGE * sizeof(T)) % 128 == 0 && (E_STAGE * 4) % 128 == 0,
                "TMA smem alignment");
  static_assert(NH == 1 || (CW == TX && TX % 8 == 0 && (HW / NV) % LXW == 0), "half tiles must be warp-aligned");
  static_assert(RA == 0 || (MINB >= 1 && NWC % 4 == 0 && RA % 8 == 0 &&
                            NWC / 4 * RA + 24 <= (NWC / 4 + 1) * MAXR), "register reallocation budget");
};

template <typename T>
struct PmlGeoT { int nx, ny, nzg, w, TN; T i2hx, i2hy, i2hz; };

// Plane-uniform constants of a z-PML cap plane seen from the inner xy footprint.
template <typename T>
struct CapCT { T ex, ezp, ezm, A, B, rB; };

// PML update of one vector row inside a z cap (inner x,y => eta(x+-1) =
// eta(y+-1) = eta_dz); same arithmetic as the naive kernel's PML branch.
template <typename T>
__device__ __noinline__ typename VecT<T>::V cap_update(typename VecT<T>::V L, typename VecT<T>::V C,
                                                       typename VecT<T>::V up, typename VecT<T>::V v,
                                                       typename VecT<T>::V xp, typename VecT<T>::V xm,
                                                       typename VecT<T>::V yp, typename VecT<T>::V ym,
                                                       typename VecT<T>::V zp, typename VecT<T>::V zm,
                                                       CapCT<T> cc, T i2hx, T i2hy, T i2hz, bool fast = false) {
  constexpr int NV = VecT<T>::N;
  T num[NV], Bd[NV], rBd[NV], res[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    const T g = add_rn(add_rn(gterm(cc.ex, cc.ex, vget(xp, c), vget(xm, c), i2hx),
                              gterm(cc.ex, cc.ex, vget(yp, c), vget(ym, c), i2hy)),
                       gterm(cc.ezp, cc.ezm, vget(zp, c), vget(zm, c), i2hz));
    num[c] = pml_num(vget(L, c), g, vget(C, c), vget(up, c), vget(v, c), cc.A);
    Bd[c] = cc.B;
    rBd[c] = cc.rB;
  }
  div_table_row<T, NV>(num, Bd, rBd, fast, res);
  return vmake<T>(res);
}

// PML path for one vector row (NV x-points at gx.., row gy, global plane kg):
// per point the Chebyshev distance d, eta on the 7-point star from the
// (w+2)-entry table (eta_{w+1} = 0 outside), the grad-eta . grad-u term and
// the damped update; points with d = 0 take the inner formula (identical
// arithmetic to the naive kernel).  Used for wall planes in / next to a cap.
// one point of the general PML path: distances dx(-1, 0, +1) along x, dy, dz
// (and their +-1 neighbours), eta on the 7-point star from the table
template <typename T>
__device__ __forceinline__ T pml_point(T Lc, T uc, T upc, T vc, T xp, T xm, T yp, T ym, T zp, T zm, int dxm,
                                       int dx, int dxp, int dy, int dym, int dyp, int dz, int dzm, int dzp,
                                       const PmlGeoT<T>& G, const T* stab, bool fast) {
  const int dxy = max(dx, dy);
  const int d = max(dxy, dz);
  if (d == 0) return upd_inner(Lc, uc, upc, vc);
  const T exp_ = stab[max(max(dxp, dy), dz)], exm = stab[max(max(dxm, dy), dz)];
  const T eyp = stab[max(max(dx, dyp), dz)], eym = stab[max(max(dx, dym), dz)];
  const T ezp = stab[max(dxy, dzp)], ezm = stab[max(dxy, dzm)];
  const T g = add_rn(add_rn(gterm(exp_, exm, xp, xm, G.i2hx), gterm(eyp, eym, yp, ym, G.i2hy)),
                     gterm(ezp, ezm, zp, zm, G.i2hz));
  return upd_pml_t(Lc, g, uc, upc, vc, stab[G.TN + d], stab[2 * G.TN + d], stab[3 * G.TN + d], fast);
}

template <typename T>
__device__ __noinline__ typename VecT<T>::V pml_row_call(typename VecT<T>::V L, typename VecT<T>::V C,
                                                         typename VecT<T>::V up, typename VecT<T>::V v,
                                                         typename VecT<T>::V xp, typename VecT<T>::V xm,
                                                         typename VecT<T>::V yp, typename VecT<T>::V ym,
                                                         typename VecT<T>::V zp, typename VecT<T>::V zm, int gx,
                                                         int gy, int kg, PmlGeoT<T> G, const T* stab, bool fast) {
  constexpr int NV = VecT<T>::N;
  const int dy = dist1(gy, G.ny, G.w), dyp = dist1(gy + 1, G.ny, G.w), dym = dist1(gy - 1, G.ny, G.w);
  const int dz = dist1(kg, G.nzg, G.w), dzp = dist1(kg + 1, G.nzg, G.w), dzm = dist1(kg - 1, G.nzg, G.w);
  int dxs[NV + 2];
#pragma unroll
  for (int c = 0; c < NV + 2; ++c) dxs[c] = dist1(gx - 1 + c, G.nx, G.w);
  T res[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c)
    res[c] = pml_point<T>(vget(L, c), vget(C, c), vget(up, c), vget(v, c), vget(xp, c), vget(xm, c), vget(yp, c),
                          vget(ym, c), vget(zp, c), vget(zm, c), dxs[c], dxs[c + 1], dxs[c + 2], dy, dym, dyp, dz,
                          dzm, dzp, G, stab, fast);
  return vmake<T>(res);
}

// Stored-eta PML path for one vector row (reading R16), with
// the eta star already staged (the eta box of the u_prev/vdt2 ring):
// e0 / exm / exp / eym / eyp / ezm / ezp are eta at the point and its 6
// neighbours (0 outside the domain, by TMA zero fill); A/B = 1 -+ eta dt from
// the point's own value computed in fp64 and rounded once; points with d = 0
// (geometric) take the inner formula.
template <typename T>
__device__ __forceinline__ typename VecT<T>::V pml_row_eta_s(
    typename VecT<T>::V L, typename VecT<T>::V C, typename VecT<T>::V up, typename VecT<T>::V v,
    typename VecT<T>::V xp, typename VecT<T>::V xm, typename VecT<T>::V yp, typename VecT<T>::V ym,
    typename VecT<T>::V zp, typename VecT<T>::V zm, int gx, int gy, int z, PmlGeoT<T> G, const float* e0,
    const float* exm, const float* exp_, const float* eym, const float* eyp, const float* ezm, const float* ezp,
    double dt) {
  constexpr int NV = VecT<T>::N;
  const int dy = dist1(gy, G.ny, G.w), dz = dist1(z, G.nzg, G.w);
  T res[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    const int d = max(max(dist1(gx + c, G.nx, G.w), dy), dz);
    const T uc = vget(C, c), upc = vget(up, c), vc = vget(v, c), Lc = vget(L, c);
    if (d == 0) {
      res[c] = upd_inner(Lc, uc, upc, vc);
    } else {
      const T g = add_rn(add_rn(gterm((T)exp_[c], (T)exm[c], vget(xp, c), vget(xm, c), G.i2hx),
                                gterm((T)eyp[c], (T)eym[c], vget(yp, c), vget(ym, c), G.i2hy)),
                         gterm((T)ezp[c], (T)ezm[c], vget(zp, c), vget(zm, c), G.i2hz));
      const double ee = (double)e0[c];
      res[c] = upd_pml(Lc, g, uc, upc, vc, (T)(1.0 - ee * dt), (T)(1.0 + ee * dt));
    }
  }
  return vmake<T>(res);
}

// ---------------------------------------------------------------------------
// Embedded wall warps (MODE_INNER_EW).  Two warps of the
// interior CTA's producer warpgroup compute the PML walls while the consumer
// warps stream the interior tile: the walls then cost SM issue slots the
// memory-bound interior leaves idle instead of whole SMs of their own.  Work
// unit = one 16 x 8 wall tile x one z-chunk, claimed from a global ticket;
// lane (warp k, lane l) owns row 4k + l/8, x points 2 (l % 8) + {0, 1}.
// Own small TMA ring (9 u stages of 24 x 16, 3 u_prev/vdt2 stages of 16 x 8),
// filled by lane 0 of wall warp 0; the register queue shifts (one plane per
// iteration, compact code: the interior's hot loop keeps the I-cache).
// Arithmetic per point is exactly the wall kernels' (column-constant /
// row-uniform fast paths on z-interior planes, pml_point elsewhere), so the
// result is bitwise the separate-launch one.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st_cs_f2(float* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float f2get(const float2& v, int c) { return c == 0 ? v.x : v.y; }
__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void ew_body(const StreamParams& P, unsigned char* ewb, const float* stab, int int_planes,
                                        int wk, int lane) {
  const StreamParams::Ew& E = P.ew;
  float* su = reinterpret_cast<float*>(ewb);
  float* sp = su + SU * EW_US;                              // [EW_SPN][u_prev | vdt2][EW_PS]
  float* sco = sp + EW_SPN * 2 * EW_PS;                      // [64 lanes][cg0, cg1, A0, A1, B0, B1, rB0, rB1]
  uint64_t* full_u = reinterpret_cast<uint64_t*>(sco + EW_COEF);
  uint64_t* empty_u = full_u + SU;
  uint64_t* full_p = empty_u + SU;
  uint64_t* empty_p = full_p + EW_SPN;
  volatile int* s_ew = reinterpret_cast<volatile int*>(empty_p + EW_SPN);   // [0] interior planes done, [1] unit
  const Coef& K = P.k;
  const int TABN = P.w + 2;
  const bool prod = wk == 0 && lane == 0;
  const int r = wk * 4 + (lane >> 3), c2 = lane & 7;
  float* myco = sco + (wk * 32 + lane) * 8;
  PmlGeoT<float> PG;
  PG.nx = P.nx; PG.ny = P.ny; PG.nzg = P.nzg; PG.w = P.w; PG.TN = TABN;
  PG.i2hx = K.i2h[0]; PG.i2hy = K.i2h[1]; PG.i2hz = K.i2h[2];
  const uint64_t pol_u = policy_evict_normal(), pol_s = policy_evict_first();
  uint32_t useq = 0, pseq = 0;                              // ring sequence numbers (persist across units)
  int cx0 = 0, ty0 = 0;
  // u plane `pl` -> ring load `n` (stage n % 9); the stage's previous use (n - 9) must be released by both warps
  auto issue_u = [&](uint32_t n, int pl) {
    const int st = (int)(n % SU);
    if (n >= (uint32_t)SU) {
      mbar_wait(&empty_u[st], ((n / SU) - 1) & 1);
      fence_proxy_async_smem();
    }
    mbar_arrive_expect_tx(&full_u[st], EW_US * 4);
    tma_load_3d(su + st * EW_US, &E.tu, &full_u[st], cx0 - R, ty0 - R, pl + R, pol_u);
    if (E.pf > 0) tma_prefetch_3d(&E.tu, cx0 - R, ty0 - R, pl + E.pf + R);
  };
  auto issue_p = [&](uint32_t n, int pl) {
    const int st = (int)(n % EW_SPN);
    if (n >= (uint32_t)EW_SPN) {
      mbar_wait(&empty_p[st], ((n / EW_SPN) - 1) & 1);
      fence_proxy_async_smem();
    }
    mbar_arrive_expect_tx(&full_p[st], 2 * EW_PS * 4);
    tma_load_3d(sp + st * 2 * EW_PS, &E.tup, &full_p[st], cx0, ty0, pl + R, pol_s);
    tma_load_3d(sp + st * 2 * EW_PS + EW_PS, &E.tv, &full_p[st], cx0, ty0, pl, pol_s);
    if (E.pf > 0) {
      tma_prefetch_3d(&E.tup, cx0, ty0, pl + E.pf + R);
      tma_prefetch_3d(&E.tv, cx0, ty0, pl + E.pf);
    }
  };

#pragma unroll 1
  while (true) {
    // ---- claim a unit (lane 0 of wall warp 0), pacing on the interior ----
    if (prod) {
      int u = -1;
#pragma unroll 1
      while (true) {
        const int rem = int_planes - s_ew[0];
        const bool last = (int)blockIdx.x >= E.last_blk;
        if (rem >= E.min_rem || (last && rem <= 0)) {
          const unsigned t = atomicAdd(E.ctr, 1u);
          u = t < (unsigned)E.nunits ? (int)t : -1;
          break;
        }
        if (!last) break;                                   // not the last wave: leave the rest to others
        __nanosleep(256);                                   // last wave: claim again once the interior is done
      }
      s_ew[1] = u;
    }
    bar_sync_n(2, 64);
    const int u = s_ew[1];
    bar_sync_n(3, 64);                                      // (s_ew[1] read by both before it is rewritten)
    if (u < 0) break;
    unsigned long long t_unit = 0;
    const bool mop = s_ew[0] >= int_planes;
    if (E.dbg && prod) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_unit));
    const int k = u / E.ntile;
    const int t = u - k * E.ntile;
    int ri = 0;
#pragma unroll 1
    while (ri + 1 < E.nreg && t >= E.reg[ri + 1].blk0) ++ri;
    const Region& g = E.reg[ri];
    const int lt = t - g.blk0;
    const int tyi = lt / g.ntx, txi = lt - tyi * g.ntx;
    cx0 = g.ax0 + txi * EW_CW;
    ty0 = g.y0 + tyi * EW_TY;
    const int zs = g.z0 + k * E.cz, ze = min(zs + E.cz, g.z1);
    const int np = ze - zs, nu = np + 2 * R;
    if (prod) {
      for (int j = 0; j < SU && j < nu; ++j) issue_u(useq + j, zs - R + j);
      for (int j = 0; j < EW_SPN && j < np; ++j) issue_p(pseq + j, zs + j);
    }
    // ---- per-lane geometry, PML coefficients -----------------------------
    const int gx = cx0 + 2 * c2, gy = ty0 + r;
    unsigned mask = 0;
#pragma unroll
    for (int c = 0; c < 2; ++c)
      if (gx + c >= g.x0 && gx + c < g.x1 && gy >= g.y0 && gy < g.y1) mask |= 1u << c;
    bool all_dx0 = true, all_dy0 = true;
#pragma unroll
    for (int c = 0; c < 2; ++c)
      if ((mask >> c) & 1u) {
        all_dx0 &= dist1(gx + c, P.nx, P.w) == 0;
        all_dy0 &= dist1(gy, P.ny, P.w) == 0;
      }
    all_dx0 = __all_sync(0xffffffffu, all_dx0);
    all_dy0 = __all_sync(0xffffffffu, all_dy0);
    const int wkind = all_dx0 ? 1 : (all_dy0 ? 2 : 0);     // 1: y-wall rows, 2: x-wall columns, 0: general
    {
      const int dy = dist1(gy, P.ny, P.w);
      const float cgy = dy == 0 ? 0.f
                                : mul_rn(sub_rn(stab[dist1(gy + 1, P.ny, P.w)], stab[dist1(gy - 1, P.ny, P.w)]),
                                         K.i2h[1]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int dx = dist1(gx + c, P.nx, P.w);
        const float cgx = dx == 0 ? 0.f
                                  : mul_rn(sub_rn(stab[dist1(gx + c + 1, P.nx, P.w)], stab[dist1(gx + c - 1, P.nx, P.w)]),
                                           K.i2h[0]);
        const int d = wkind == 1 ? dy : dx;
        myco[c] = wkind == 1 ? cgy : cgx;
        myco[2 + c] = stab[TABN + d];
        myco[4 + c] = stab[2 * TABN + d];
        myco[6 + c] = stab[3 * TABN + d];
      }
    }
    // ---- warm-up: planes zs-4 .. zs+3 -> queue ------------------------------
    const int own = (r + R) * EW_SW + R + 2 * c2;          // my centre in a u stage
    float2 q[2 * R + 1];
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) {
      const uint32_t n = useq + j;
      mbar_wait(&full_u[n % SU], (n / SU) & 1);
      q[j] = lds2(su + (n % SU) * EW_US + own);
    }
    __syncwarp();
#pragma unroll 1
    for (int j = 0; j < R; ++j) {                           // planes zs-4..zs-1: only their own rows were needed
      if (lane == 0) mbar_arrive(&empty_u[(useq + j) % SU]);
      if (prod && j + SU < nu) issue_u(useq + j + SU, zs - R + j + SU);
    }
    float* optr = static_cast<float*>(P.out) + (int64_t)(zs + R) * P.plane + (int64_t)gy * P.pitch + gx;
    const bool fast = P.fastdiv != 0;
    // ---- planes -------------------------------------------------------------
#pragma unroll 1
    for (int i = 0; i < np; ++i) {
      const int z = zs + i;
      {
        const uint32_t n = useq + i + 2 * R;                // leading plane z + 4
        mbar_wait(&full_u[n % SU], (n / SU) & 1);
        q[2 * R] = lds2(su + (n % SU) * EW_US + own);
      }
      const int sc = (int)((useq + i + R) % SU);            // centre plane z
      const float* S = su + sc * EW_US + own;
      float2 Y[2 * R + 1];
#pragma unroll
      for (int jj = 0; jj <= 2 * R; ++jj) Y[jj] = jj == R ? q[R] : lds2(S + (jj - R) * EW_SW);
      const float2 xl0 = lds2(S - 4), xl1 = lds2(S - 2), xr0 = lds2(S + 2), xr1 = lds2(S + 4);
      const float Xv[10] = {xl0.x, xl0.y, xl1.x, xl1.y, q[R].x, q[R].y, xr0.x, xr0.y, xr1.x, xr1.y};
      const uint32_t pn = pseq + i;
      const int spp = (int)(pn % EW_SPN);
      mbar_wait(&full_p[spp], (pn / EW_SPN) & 1);
      const float2 upv = lds2(sp + spp * 2 * EW_PS + r * EW_CW + 2 * c2);
      const float2 vv = lds2(sp + spp * 2 * EW_PS + EW_PS + r * EW_CW + 2 * c2);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_u[sc]);
        mbar_arrive(&empty_p[spp]);
      }
      if (prod) {
        if (i + R + SU < nu) issue_u(useq + i + R + SU, z + SU);
        if (i + EW_SPN < np) issue_p(pn + EW_SPN, z + EW_SPN);
      }
      float L[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        L[c] = mul_rn(K.c0, Xv[4 + c]);
#pragma unroll
        for (int m = 1; m <= R; ++m) L[c] = fma_rn(K.cx[m - 1], add_rn(Xv[4 + c + m], Xv[4 + c - m]), L[c]);
#pragma unroll
        for (int m = 1; m <= R; ++m) L[c] = fma_rn(K.cy[m - 1], add_rn(f2get(Y[R + m], c), f2get(Y[R - m], c)), L[c]);
#pragma unroll
        for (int m = 1; m <= R; ++m) L[c] = fma_rn(K.cz[m - 1], add_rn(f2get(q[R + m], c), f2get(q[R - m], c)), L[c]);
      }
      const int kg = z + P.zoff;
      float o[2];
      if (wkind != 0 && kg > P.w && kg < P.nzg - P.w - 1) {
        const float4 c0 = *reinterpret_cast<const float4*>(myco), c1 = *reinterpret_cast<const float4*>(myco + 4);
        const float cg[2] = {c0.x, c0.y}, A[2] = {c0.z, c0.w};
        float num[2];
        const float Bd[2] = {c1.x, c1.y}, rBd[2] = {c1.z, c1.w};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float gd = wkind == 2 ? mul_rn(cg[c], mul_rn(sub_rn(Xv[5 + c], Xv[3 + c]), K.i2h[0]))
                                      : mul_rn(cg[c], mul_rn(sub_rn(f2get(Y[R + 1], c), f2get(Y[R - 1], c)), K.i2h[1]));
          num[c] = pml_num(L[c], gd, Xv[4 + c], f2get(upv, c), f2get(vv, c), A[c]);
        }
        div_table_row<float, 2>(num, Bd, rBd, fast, o);
      } else {
        const int dy = dist1(gy, P.ny, P.w), dym = dist1(gy - 1, P.ny, P.w), dyp = dist1(gy + 1, P.ny, P.w);
        const int dz = dist1(kg, P.nzg, P.w), dzm = dist1(kg - 1, P.nzg, P.w), dzp = dist1(kg + 1, P.nzg, P.w);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          o[c] = pml_point<float>(L[c], Xv[4 + c], f2get(upv, c), f2get(vv, c), Xv[5 + c], Xv[3 + c],
                                  f2get(Y[R + 1], c), f2get(Y[R - 1], c), f2get(q[R + 1], c), f2get(q[R - 1], c),
                                  dist1(gx + c - 1, P.nx, P.w), dist1(gx + c, P.nx, P.w),
                                  dist1(gx + c + 1, P.nx, P.w), dy, dym, dyp, dz, dzm, dzp, PG, stab, fast);
      }
      if (mask == 3u) {
        st_cs_f2(optr, make_float2(o[0], o[1]));
      } else {
        if (mask & 1u) optr[0] = o[0];
        if (mask & 2u) optr[1] = o[1];
      }
      // fused halo exchange of edge planes (both targets independent, as in stream_body)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        float* rbase = nullptr;
        if (side == 0 && z < R && P.rlo) rbase = static_cast<float*>(P.rlo) + (int64_t)z * P.plane;
        if (side == 1 && z >= P.nzl - R && P.rhi) rbase = static_cast<float*>(P.rhi) + (int64_t)(z - (P.nzl - R)) * P.plane;
        if (rbase) {
          float* rp = rbase + (int64_t)gy * P.pitch + gx;
          if (mask & 1u) rp[0] = o[0];
          if (mask & 2u) rp[1] = o[1];
        }
      }
      optr += P.plane;
#pragma unroll
      for (int j = 0; j < 2 * R; ++j) q[j] = q[j + 1];
    }
    // the last 4 loads (planes ze..ze+3) were only ever leading planes: release
    // them so the ring can be refilled for the next unit
    __syncwarp();
    if (lane == 0)
      for (int j = np + R; j < nu; ++j) mbar_arrive(&empty_u[(useq + j) % SU]);
    useq += nu;
    pseq += np;
    if (E.dbg && prod) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      atomicAdd(E.dbg + (mop ? 2 : 0), t1 - t_unit);
      atomicAdd(E.dbg + (mop ? 3 : 1), (unsigned long long)np);
      atomicAdd(E.dbg + (mop ? 5 : 4), 1ull);
    }
  }
  // every CTA's wall warps finish exactly once; the last one re-arms the ticket
  // for the next launch (no claim can follow: all CTAs have made their last)
  if (prod) {
    __threadfence();
    if (atomicAdd(E.ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(E.ctr, 0u);
      atomicExch(E.ctr + 1, 0u);
    }
  }
}

// The body of one work unit (tile x z-chunk) of k_stream; `unit0` = its index
// in the launch's region list (blockIdx.x for k_stream, remapped by k_mix).
// CL > 1 (interior only, TY = 2R): CL CTAs of a thread-block cluster hold CL
// vertically adjacent tiles.  Their u windows overlap by 2R rows, so each u
// stage is assembled from (2R)-row boxes: box k (rows [y0_k - R, y0_k + R) of
// CTA k's tile) is loaded ONCE by CTA k and multicast into CTAs k-1 and k
// (TMA .multicast::cluster); the last CTA also loads the bottom box.  A box
// lands at the same shared-memory offset in every destination, half k & 1 of
// the stage, so odd CTAs see their window with its two halves swapped (the
// consumers' row offsets absorb it).  A stage may be refilled only when the
// consumers of both destination CTAs released it: every consumer warp also
// arrives on the next CTA's empty barrier.  The shared halo rows of y-adjacent
// tiles are thus read from L2/DRAM once and the pair streams in lockstep.
template <int TX, int CW, int TY, int TYT, int MODE, int MINB, int RA = 0, typename T = float, int PAIR = 0,
          int CL = 1>
__device__ __forceinline__ void
stream_body(const CUtensorMap& tm_u,    // u^n, box (HW+8, TY+8, 1)
            const CUtensorMap& tm_up,   // u^{n-1}, box (CW, TY, 1)
            const CUtensorMap& tm_v,    // vdt2, box (CW, TY, 1)
            const StreamParams& P, const int unit0) {
  constexpr bool EW = MODE == MODE_INNER_EW;               // embedded wall warps
  constexpr bool INN = MODE == MODE_INNER || EW;             // interior update in the consumer warps
  using C = StreamCfg<TX, CW, TY, TYT, MINB, RA, T, MODE == MODE_WALL_ETA, EW ? EW_BYTES : 0>;
  static_assert(!EW || (sizeof(T) == 4 && RA == EW_RC && PAIR == 0 && CL == 1 && C::NWC % 4 == 0 &&
                        C::NWC / 4 * EW_RC + EW_RP <= (C::NWC / 4 + 1) * C::MAXR),
                "embedded walls: fp32 interior with a producer warpgroup of 4 warps (TMA + 2 wall warps + 1)");
  using V = typename VecT<T>::V;
  constexpr int NV = C::NV;
  static_assert(CL == 1 || (MODE == MODE_INNER && C::NH == 1 && TY == 2 * R && TYT == 1 && PAIR == 0 && CL <= 8),
                "cluster multicast: interior tiles of 2R rows, one u box per half");
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  constexpr int KX = (R + NV - 1) / NV;           // x-neighbour vectors on each side
  constexpr int XC = KX * NV;                     // index of the first centre point in X[]
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  // (swizzled u stages: the layout starts at the next 1024-B boundary)
  unsigned char* smem_raw = smem_dyn + (C::SWZ ? ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u) : 0u);
  T* su = reinterpret_cast<T*>(smem_raw);
  T* sup = su + SU * C::U_STAGE;
  T* sv = sup + C::SPN * C::P_STAGE;
  float* se = reinterpret_cast<float*>(smem_raw + C::E_OFF);   // stored-eta ring (MODE_WALL_ETA)
  uint64_t* full_u = reinterpret_cast<uint64_t*>(smem_raw + C::BAR_OFF);
  uint64_t* empty_u = full_u + SU;
  uint64_t* full_p = empty_u + SU;
  uint64_t* empty_p = full_p + C::SPN;
  T* stab = reinterpret_cast<T*>(smem_raw + C::TAB_OFF);
  const int TABN = P.w + 2;
  // PAIR step 1: per-publication arrival counts of the consumer warps, in a ring
  // of 16 (warps drift by at most ~10 planes: the 9-stage u ring couples them)
  __shared__ unsigned s_arr[PAIR ? 16 : 1];

  // ---- work unit ---------------------------------------------------------
  // PAIR: work units are handed out by a ticket counter in CTA start order, so
  // a step-2 unit only ever waits on units already taken by running (or
  // finished) CTAs -- deadlock-free whatever order the hardware dispatches in
  int unit = unit0;
  if (PAIR) {
    __shared__ int s_unit;
    if (threadIdx.x == 0) s_unit = (int)atomicAdd(P.prog + P.pair_ticket, 1u);
    __syncthreads();
    unit = s_unit;
  }
  int b = unit, ri = 0;
  if (P.inter2) {
    ri = unit & 1;
    b = (unit >> 1) + P.reg[ri].blk0;
  } else {
#pragma unroll 1
    while (ri + 1 < P.nreg && b >= P.reg[ri + 1].blk0) ++ri;
  }
  const Region& G = P.reg[ri];
  b -= G.blk0;
  const int ncol = G.ntx * G.nty;
  int zc = b / ncol;
  const int rem = b - zc * ncol;
  int tyi, txi;
  int role = 0;                          // PAIR: 1 = step 1, 2 = step 2
  if (PAIR) {
    // groups of one tile row each, in dependency order (S1 r+1 before S2 r)
    const int g = unit / G.ntx, code = P.pair_groups[g];
    role = code >> 28;
    zc = (code >> 16) & 0xfff;
    tyi = code & 0xffff;
    txi = unit - g * G.ntx;
  } else if (CL > 1) {                     // clusters of CL tile rows, consecutive blocks = one cluster
    const int pr = rem / (G.ntx * CL);
    const int r2 = rem - pr * G.ntx * CL;
    txi = r2 / CL;
    tyi = pr * CL + (r2 - txi * CL);         // r2 % CL == %cluster_ctarank (blk0, ncol multiples of CL)
  } else if (P.order < 0) {                // bands of -order tile rows, x-major inside a band
    const int bh = -P.order;
    const int band = rem / (bh * G.ntx);
    const int bsz = min(bh, G.nty - band * bh);
    const int r2 = rem - band * bh * G.ntx;
    txi = r2 / bsz;
    tyi = band * bh + (r2 - txi * bsz);
  } else if (P.order == 0) {
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
  int zs = G.z0 + zc * P.cz;
  int ze = min(zs + P.cz, G.z1);
  // PAIR step 2: chunk k covers planes [k cz - 4, (k+1) cz - 4), so that it
  // needs only step-1 chunks <= k (scheduled before it: no deadlock)
  if (PAIR && role == 2) {
    zs = max(zs - R, G.z0);
    ze = ze >= G.z1 ? G.z1 : ze - R;
  }

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;

  // ---- setup: barriers, PML tables --------------------------------------
  if (tid == 0) {
    prefetch_tmap(P.gu ? P.gu : &tm_u);
    prefetch_tmap(P.gup ? P.gup : &tm_up);
    prefetch_tmap(P.gv ? P.gv : &tm_v);
#pragma unroll
    // cluster: box k feeds CTAs k-1 and k, so CTA k refills a stage after both released it
    for (int s = 0; s < SU; ++s) { mbar_init(&full_u[s], 1); mbar_init(&empty_u[s], C::NWC * (crank > 0 ? 2 : 1)); }
#pragma unroll
    for (int s = 0; s < C::SPN; ++s) { mbar_init(&full_p[s], 1); mbar_init(&empty_p[s], C::NWC); }
    if (EW) {
      uint64_t* eb = reinterpret_cast<uint64_t*>(smem_raw + C::EW_OFF + (SU * EW_US + 2 * EW_SPN * EW_PS + EW_COEF) * 4);
      for (int s = 0; s < SU; ++s) { mbar_init(&eb[s], 1); mbar_init(&eb[SU + s], 2); }
      for (int s = 0; s < EW_SPN; ++s) { mbar_init(&eb[2 * SU + s], 1); mbar_init(&eb[2 * SU + EW_SPN + s], 2); }
      int* sew = reinterpret_cast<int*>(eb + 2 * (SU + EW_SPN));
      sew[0] = 0;
      sew[1] = -1;
      prefetch_tmap(&P.ew.tu);
      prefetch_tmap(&P.ew.tup);
      prefetch_tmap(&P.ew.tv);
    }
    fence_mbar_init();
  }
  for (int i = tid; i < 4 * TABN; i += C::NT) stab[i] = static_cast<const T*>(P.tab)[i];
  if (PAIR && tid < 16) s_arr[tid] = 0;
  __syncthreads();
  if (CL > 1) cluster_sync_all();            // peers' barriers initialised before any multicast / remote arrive

  // ======================= producer warp =================================
  if (wid >= C::NWC) {
    // the cluster producer (multicast masks, remote barriers) needs 32 registers;
    // the budget 4 x 112 + 32 = 5 x 96 still holds for the interior tile
    if (EW) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(EW_RP) : "memory");
      if (wid == C::NWC + 1 || wid == C::NWC + 2) {       // the wall warps
        ew_body(P, smem_raw + C::EW_OFF, reinterpret_cast<const float*>(stab), ze - zs, wid - C::NWC - 1, lane);
        return;
      }
    } else if (RA > 0 && CL > 1) {
      static_assert(CL == 1 || C::NWC / 4 * RA + 32 <= (C::NWC / 4 + 1) * C::MAXR, "cluster producer registers");
      asm volatile("setmaxnreg.dec.sync.aligned.u32 32;" ::: "memory");
    } else if (RA > 0) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
    }
    auto produce = [&]() {
    const uint64_t pol_u = P.upol ? policy_evict_normal() : policy_evict_last();  // u^n: halo re-reads
    // u^{n-1}, vdt2: streamed once -- except in a PAIR step-1 block, whose
    // u^{n-1} (overwritten by u^{n+1}) and vdt2 lines step 2 reads again
    // (evict_last here and on the u^{n+1} stores measured no different, §5h)
    const uint64_t pol_s = (PAIR && role == 1) ? policy_evict_normal() : policy_evict_first();
    const CUtensorMap* mu = (PAIR && role == 2) ? P.gu2 : (P.gu ? P.gu : &tm_u);
    const CUtensorMap* mup = (PAIR && role == 2) ? P.gup2 : (P.gup ? P.gup : &tm_up);
    const CUtensorMap* mv = P.gv ? P.gv : &tm_v;
    // PAIR step 2: u^{n+1} plane p may be loaded once the step-1 blocks of this
    // tile and of its x/y neighbours have stored it (release/acquire on the
    // progress counters, then a generic->async proxy fence for the TMA read)
    // counters: prog[k * ntile + tile] = planes of step-1 chunk k stored for the
    // tile.  Neighbour counters (absent neighbours read the tile's own) are polled
    // together; `known` = their minimum at the last poll of chunk kcur, so most
    // planes need no poll at all
    const int tile = tyi * G.ntx + txi, ntile = G.ntx * G.nty;
    const int nbt[5] = {tile, txi > 0 ? tile - 1 : tile, txi + 1 < G.ntx ? tile + 1 : tile,
                        tyi > 0 ? tile - G.ntx : tile, tyi + 1 < G.nty ? tile + G.ntx : tile};
    unsigned known = 0;
    int kcur = -1;
    unsigned long long dbg_t0 = 0, dbg_slack = 0;
    unsigned dbg_polls = 0, dbg_fails = 0;
    if (PAIR && (P.pair_dbg & 8)) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t0));
    auto wait_plane = [&](int p) {
      if (!PAIR || role != 2 || p < 0 || p >= P.nzl || (P.pair_dbg & 1)) return;
      const int kp = p / P.cz;
      const unsigned need = (unsigned)(p - kp * P.cz + 1);
      if (kp != kcur) { kcur = kp; known = 0; }
      if (known >= need) return;
      const unsigned* base = P.prog + (int64_t)kp * ntile;
      unsigned long long spins = 0;
#pragma unroll 1
      while (true) {
        unsigned v[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) v[k] = ld_acquire_gpu_u32(base + nbt[k]);
        known = min(min(min(v[0], v[1]), min(v[2], v[3])), v[4]);
        if (P.pair_dbg & 8) { ++dbg_polls; if (known < need) ++dbg_fails; else dbg_slack += known - need; }
        if (known >= need) break;
        __nanosleep(32);
        if (++spins > (1ull << 27)) __trap();       // a missing producer: fail, never hang
      }
      fence_proxy_async_global();
    };
    // u plane p (local z, p >= zs-4) lives in u stage (p - zs + 4) % 9, use (p - zs + 4) / 9
    auto issue_u = [&](int p, int st) {
      wait_plane(p);
      mbar_arrive_expect_tx(&full_u[st], C::U_STAGE * sizeof(T));
      if (CL > 1) {
        // box crank (my window's top half) -> CTAs crank-1 and crank; the last
        // CTA also loads the bottom box (its window's bottom half) for itself
        constexpr int HR = 2 * R * C::SW;      // elements per (2R)-row half
        const uint16_t mask = (uint16_t)((1u << crank) | (crank > 0 ? 1u << (crank - 1) : 0u));
        tma_load_3d_mc(su + st * C::U_STAGE + (crank & 1) * HR, mu, &full_u[st], bx0 - R, ty0 - R, p + R, mask,
                       pol_u);
        if (crank == CL - 1)
          tma_load_3d(su + st * C::U_STAGE + ((crank + 1) & 1) * HR, mu, &full_u[st], bx0 - R, ty0 + R, p + R,
                      pol_u);
      } else {
#pragma unroll
        for (int h = 0; h < C::NH; ++h)
          tma_load_3d(su + st * C::U_STAGE + h * C::U_HALF, mu, &full_u[st], bx0 + h * C::HW - R, ty0 - R, p + R,
                      pol_u);
      }
    };
    // p plane p (p >= zs) lives in p stage (p - zs) % 3, use (p - zs) / 3
    auto issue_p = [&](int p, int st) {
      // (the eta box delivers EW x (TY+2) floats; E_STAGE is that rounded up for alignment)
      mbar_arrive_expect_tx(&full_p[st], 2 * C::P_STAGE * sizeof(T) + (MODE == MODE_WALL_ETA ? C::EW * (TY + 2) * 4 : 0));
      tma_load_3d(sup + st * C::P_STAGE, mup, &full_p[st], cx0, ty0, p + R, pol_s);
      tma_load_3d(sv + st * C::P_STAGE, mv, &full_p[st], cx0, ty0, p, pol_s);
      if (MODE == MODE_WALL_ETA) tma_load_3d(se + st * C::E_STAGE, &P.tm_eta, &full_p[st], cx0 - 4, ty0 - 1, p, pol_s);
    };
    for (int s = 0; s < SU; ++s)
      if (zs - R + s <= ze + R - 1) issue_u(zs - R + s, s);      // planes zs-4 .. zs+4
    for (int s = 0; s < C::SPN; ++s)
      if (zs + s < ze) issue_p(zs + s, s);                       // planes zs .. zs+2
    // refill in release order: when plane t is released, u plane t+9 and p plane t+3 go in
#pragma unroll 1
    for (int t = zs - R; t + SU <= ze + R - 1 || t + C::SPN < ze; ++t) {
      if (t + SU <= ze + R - 1) {
        const int o = t - zs + R;
        // the consumers' generic-proxy reads of this stage are ordered before
        // the TMA (async-proxy) overwrite: mbarrier release/acquire + proxy fence
        // (cluster: the previous CTA's consumers released it too, and the
        // multicast also overwrites their copy)
        if (CL > 1 && P.pair_dbg == 16) {     // (A/B: cluster-scope acquire + full proxy fence)
          mbar_wait_cluster(&empty_u[o % SU], (o / SU) & 1);
          fence_proxy_async_all();
        } else {
          mbar_wait(&empty_u[o % SU], (o / SU) & 1);
          fence_proxy_async_smem();
        }
        issue_u(t + SU, o % SU);
      }
      if (t >= zs && t + C::SPN < ze) {
        const int o = t - zs;
        mbar_wait(&empty_p[o % C::SPN], (o / C::SPN) & 1);
        fence_proxy_async_smem();
        issue_p(t + C::SPN, o % C::SPN);
      }
      if (P.pf > 0) {
        const int pu = t + SU + P.pf, pp = t + C::SPN + P.pf;
        if (pu <= ze + R - 1) {
#pragma unroll
          for (int h = 0; h < C::NH; ++h) tma_prefetch_3d(mu, bx0 + h * C::HW - R, ty0 - R, pu + R);
          if (CL > 1 && crank == CL - 1) tma_prefetch_3d(mu, bx0 - R, ty0 + R, pu + R);
        }
        if (t >= zs && pp < ze) {
          tma_prefetch_3d(mup, cx0, ty0, pp + R);
          tma_prefetch_3d(mv, cx0, ty0, pp);
        }
      }
    }
    if (PAIR && (P.pair_dbg & 8)) {          // timeline record after the counters (timing probe)
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* rec = reinterpret_cast<unsigned long long*>(P.prog + P.pair_dbg_off) + 6 * unit;
      rec[0] = ((unsigned long long)role << 48) | ((unsigned long long)zc << 32) | ((unsigned)tyi << 16) | txi;
      rec[1] = smid;
      rec[2] = dbg_t0;
      rec[3] = t1;
      rec[4] = ((unsigned long long)dbg_polls << 32) | dbg_fails;
      rec[5] = dbg_slack;
    }
    };
    if (CL > 1) {
      // every thread stays to the final cluster barrier (peers still arrive on our barriers)
      if (wid == C::NWC && lane == 0) produce();
      __syncwarp();
      cluster_sync_all();
      return;
    }
    if (wid != C::NWC || lane != 0) return;
    produce();
    return;
  }

  // ======================= consumer warps ================================
  if (RA > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(RA) : "memory");
  const int lx = (wid % C::WX) * C::LXW + (lane % C::LXW);
  // swizzled x-wall stages: a warp's 8 rows are read 2 per quarter-warp (LDS.128
  // phases of 8 lanes); with the 128-B swizzle (chunk ^= row & 7) rows r and r+1
  // overlap in 2 of their 4 chunks, rows r and r+4 are disjoint -- so a quarter
  // takes rows {q, q+4}
  const int lrow = lane / C::LXW;
  const int ly = (wid / C::WX) * C::LYW +
                 ((C::SWZ && C::LYW == 8) ? ((lrow >> 1) | ((lrow & 1) << 2)) : lrow);
  const int gx = cx0 + NV * lx;             // first x of my vector
  const int gy = ty0 + ly * TYT;            // first y of my rows
  // the global point coordinates of my vector: (px + c, py + r); for seams the
  // right-wall half (seam columns [0, w)) lies on row t - 1 at x = nx - w + col,
  // the left-wall half on row t at x = col - w
  constexpr bool SEAM = MODE == MODE_SEAM;
  static_assert(!SEAM || (TYT == 1 && true), "seam tiles: one row per lane");
  const int scol = gx - G.x0;
  const bool sright = SEAM && scol < P.w;
  const int px = SEAM ? (sright ? P.nx - P.w + scol : scol - P.w) : gx;
  const int py = SEAM ? gy - (sright ? 1 : 0) : gy;
  // smem offsets (elements) of my vector in row 0 of the tile, u stage / p stage
  const int hf = (NV * lx) / C::HW;         // which half box (warp-uniform)
  // element offset of logical window row l (0 .. TY+2R-1 of the u box) at my
  // column inside a u stage; in an odd-rank cluster CTA the two (2R)-row halves
  // of the window are swapped (the multicast layout, see above)
  // (l ^ 2R) = (l + 2R) mod 4R for l in [0, 4R): computed per use from one
  // register (rematerialised rather than holding 9 offsets live in the loop)
  const int colo = hf * C::U_HALF + cxo + NV * lx - hf * C::HW + R;
  const int lyf = ly * TYT + (CL > 1 ? (crank & 1) * 2 * R : 0);
  auto yo = [&](int jj) -> int {
    return colo + (CL > 1 ? ((lyf + jj) & (4 * R - 1)) : (lyf + jj)) * C::SW;
  };
  const int uo = yo(R);                     // my first own row
  // swizzled stages (C::SWZ): element offset of the float4 chunk `ch` of box row `rr`
  const int kc = (cxo + NV * lx + R) / NV;  // my centre chunk
  auto uz = [&](int rr, int ch) -> int { return rr * C::SW + ((ch ^ (rr & 7)) * NV); };
  // my centre-chunk column of window rows ly*TYT + j, j = 0..7 (row j+8 repeats
  // row j), packed 3 bits per row in one register (9 hoisted offsets spilled)
  unsigned zsw = 0;
  if (C::SWZ) {
#pragma unroll
    for (int j = 0; j < 8; ++j) zsw |= (unsigned)((kc ^ ((ly * TYT + j) & 7)) & 7) << (3 * j);
  }
  auto uzc = [&](int jj) -> int {             // u-stage offset of window row ly*TYT + jj, my centre chunk
    return (ly * TYT + jj) * C::SW + (int)((zsw >> (3 * (jj & 7))) & 7u) * NV;
  };
  const int po = (ly * TYT) * CW + NV * lx;

  // ---- per-thread geometry: store mask, PML coefficients -----------------
  unsigned mask = 0;                         // bit (r*NV + c): point is in the region
#pragma unroll
  for (int r = 0; r < TYT; ++r)
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      const int x = gx + c, y = gy + r;
      if (x >= G.x0 && x < G.x1 && y >= G.y0 && y < G.y1 && (!SEAM || (py + r >= 0 && py + r < P.ny)))
        mask |= 1u << (r * NV + c);
    }
  if (NV * lx >= CW) mask = 0;               // phantom lane beyond the computed width
  const bool full = mask == (TYT * NV == 32 ? 0xffffffffu : ((1u << (TYT * NV)) - 1u));
  const CoefT<T>& K = coef_of<T>(P);
  PmlGeoT<T> PG;
  PG.nx = P.nx; PG.ny = P.ny; PG.nzg = P.nzg; PG.w = P.w; PG.TN = TABN;
  PG.i2hx = K.i2h[0]; PG.i2hy = K.i2h[1]; PG.i2hz = K.i2h[2];
  // fused mode: does any in-region point of my warp lie in the x/y PML?
  bool warp_xy_pml = false;
  if (MODE == MODE_FUSED) {
    bool mine = false;
#pragma unroll
    for (int r = 0; r < TYT; ++r)
#pragma unroll
      for (int c = 0; c < NV; ++c)
        if ((mask >> (r * NV + c)) & 1u)
          mine |= dist1(gx + c, P.nx, P.w) > 0 || dist1(gy + r, P.ny, P.w) > 0;
    warp_xy_pml = __any_sync(0xffffffffu, mine);
  }
  // wall mode, planes with dz(k-1) = dz(k) = dz(k+1) = 0: a warp whose points
  // all have dx = 0 (y wall away from the corners) has a row-uniform eta star
  // (grad eta = d_y eta only); one whose points all have dy = 0 (x wall) a
  // column-constant one (d_x eta only).  Precompute those coefficients once:
  //   cg = (eta(+e_a) - eta(-e_a)) / (2 h_a), A_d, B_d
  // Warps mixing both (corners) take the general path.
  // The coefficients live in small per-CTA shared tables (cg, A, B per tile
  // column / row), re-read inside the specialised branches each plane: kept in
  // registers across the loop they were spilled to local memory around the
  // general path's call, and the LDL latency stalled the wall kernels (§5).
  int wkind = 0;                             // 1: y-wall rows, 2: x-wall columns, 0: general
  constexpr bool WALLS = MODE == MODE_WALL || MODE == MODE_WALLX || MODE == MODE_WALLY || MODE == MODE_SEAM;
  constexpr bool WT = WALLS || MODE == MODE_FUSED;
  __shared__ __align__(16) T s_wc[WT ? 4 * CW : 1];   // per column: cg_x, A, B, RN(1/B)
  __shared__ __align__(16) T s_wr[WT ? 4 * TY : 1];   // per row: cg_y, A, B, RN(1/B)
  const int wci = min(NV * lx, CW - NV);     // my first table column (phantom lanes clamp)
  // fused mode: warps touching the x/y PML take the same specialised paths
  const bool wallw = WALLS || MODE == MODE_WALL_ETA || (MODE == MODE_FUSED && warp_xy_pml);
  if (WALLS || MODE == MODE_FUSED) {
    bool all_dx0 = true, all_dy0 = true;
#pragma unroll
    for (int r = 0; r < TYT; ++r)
#pragma unroll
      for (int c = 0; c < NV; ++c)
        if ((mask >> (r * NV + c)) & 1u) {
          all_dx0 &= dist1(px + c, P.nx, P.w) == 0;
          all_dy0 &= dist1(py + r, P.ny, P.w) == 0;
        }
    all_dx0 = __all_sync(0xffffffffu, all_dx0);
    all_dy0 = __all_sync(0xffffffffu, all_dy0);
    wkind = all_dx0 ? 1 : (all_dy0 ? 2 : 0);
    if ((MODE == MODE_WALLX || SEAM) && wkind == 1) wkind = 0;   // (not compiled in this kernel: general path)
    if (MODE == MODE_WALLY && wkind == 2) wkind = 0;
    // an inner point (d = 0) inside a wall region (the frames of a two-step
    // pair reach 4 or 8 cells into the inner box) takes cg = 0, A = B = 1:
    // ((2u - up) + v (L + 0)) / 1, bitwise the inner update (up to the sign of 0)
    if (lx == 0) {                           // one writer per tile row
#pragma unroll
      for (int r = 0; r < TYT; ++r) {
        const int dy = dist1(gy + r, P.ny, P.w);
        s_wr[ly * TYT + r] =
            dy == 0 ? T(0)
                    : mul_rn(sub_rn(stab[dist1(gy + r + 1, P.ny, P.w)], stab[dist1(gy + r - 1, P.ny, P.w)]),
                             PG.i2hy);
        s_wr[TY + ly * TYT + r] = stab[TABN + dy];
        s_wr[2 * TY + ly * TYT + r] = stab[2 * TABN + dy];
        s_wr[3 * TY + ly * TYT + r] = stab[3 * TABN + dy];
      }
    }
    if (ly == 0 && NV * lx < CW) {           // one writer per tile column
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        const int dx = dist1(px + c, P.nx, P.w);
        s_wc[NV * lx + c] =
            dx == 0 ? T(0)
                    : mul_rn(sub_rn(stab[dist1(px + c + 1, P.nx, P.w)], stab[dist1(px + c - 1, P.nx, P.w)]),
                             PG.i2hx);
        s_wc[CW + NV * lx + c] = stab[TABN + dx];
        s_wc[2 * CW + NV * lx + c] = stab[2 * TABN + dx];
        s_wc[3 * CW + NV * lx + c] = stab[3 * TABN + dx];
      }
    }
    // consumer warps only (the producer warps have left): named barrier 1
    asm volatile("bar.sync 1, %0;" ::"r"(C::NWC * 32) : "memory");
  }
  // (seams: both halves of seam t sit at t * pitch + gx - (x0 + w) when a row
  // is exactly nx = pitch elements long; the host guarantees that)
  const int64_t sadj = SEAM ? -(int64_t)(G.x0 + P.w) : 0;
  T* optr = static_cast<T*>((PAIR && role == 2) ? P.out2 : P.out) + (int64_t)(zs + R) * P.plane +
            (int64_t)gy * P.pitch + gx + sadj;
  // seams: the window row of my half that is not a grid row (row -1 of the
  // right half, row ny of the left half) must read as 0 (the Dirichlet fringe),
  // and the x neighbours across the seam boundary too
  const int yzero = !SEAM ? -100 : (sright ? R - gy : P.ny - gy + R);   // window index jj, or out of range
  // (only warps within R seams of either end mask: a warp-uniform branch)
  const bool yzero_warp = SEAM && __any_sync(0xffffffffu, yzero >= 0 && yzero < TYT + 2 * R);
  const bool xr_zero = SEAM && scol + NV == P.w;   // right half's last vector: x+1.. beyond nx-1
  const bool xl_zero = SEAM && scol == P.w;        // left half's first vector: x-1.. below 0
  // PAIR: the source cell is injected by the block that computes it (step 1
  // adds inc[n], step 2 inc[n+1]); -1 if not in my vector rows
  int src_r = -1, src_c = 0;
  if (PAIR && P.src_k >= 0) {
#pragma unroll
    for (int r = 0; r < TYT; ++r)
      if (gy + r == P.src_j && P.src_i >= gx && P.src_i < gx + NV && ((mask >> (r * NV + P.src_i - gx)) & 1u)) {
        src_r = r;
        src_c = P.src_i - gx;
      }
  }

  // cluster: the next CTA's empty_u barriers (its box lands in my stages)
  const uint32_t rem_empty = (CL > 1 && crank < CL - 1) ? mapa_shared(empty_u, crank + 1) : 0u;

  // stored eta staged through the u_prev/vdt2 ring: my points' eta of the
  // previous plane is carried in registers (its stage is already released)
  constexpr bool ES = MODE == MODE_WALL_ETA;
  float eprev[ES ? TYT : 1][ES ? NV : 1];
  if (ES) {
#pragma unroll
    for (int r = 0; r < TYT; ++r)
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        const int x = gx + c, y = gy + r, zz = zs - 1;
        eprev[r][c] = (zz >= 0 && x < P.nx && y < P.ny) ? __ldg(P.eta + ((int64_t)zz * P.ny + y) * P.pitch + x) : 0.f;
      }
  }

  // ---- warm-up: planes zs-4 .. zs+3 (stages 0..7, first use) -> queue ----
  V q[9][TYT];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    mbar_wait(&full_u[s], 0);
#pragma unroll
    for (int r = 0; r < TYT; ++r)
      q[s][r] = ldv(su + s * C::U_STAGE + (C::SWZ ? uzc(R + r) : uo + r * C::SW));
  }
  __syncwarp();
  if (lane == 0) {                           // planes zs-4..zs-1 are not needed again
#pragma unroll
    for (int s = 0; s < R; ++s) {
      mbar_arrive(&empty_u[s]);
      if (CL > 1 && crank < CL - 1) mbar_arrive_remote(rem_empty + 8 * s);   // its box is in my stage
    }
  }

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
      for (int r = 0; r < TYT; ++r)
        q[sl][r] = ldv(su + sl * C::U_STAGE + (C::SWZ ? uzc(R + r) : uo + r * C::SW));

      // 2. Laplacian of all NV*TYT points (interleaved chains)
      const T* S = su + sc * C::U_STAGE + uo;
      // swizzled stages: re-derive the row offsets from the packed register
      // every plane (hoisted, the 9 offsets would spill)
      int kcv = kc;
      if (C::SWZ) asm volatile("" : "+r"(zsw), "+r"(kcv));
      V Y[TYT + 2 * R];                      // rows -4 .. TYT+3 at my vector
#pragma unroll
      for (int jj = 0; jj < TYT + 2 * R; ++jj) {
        if (jj >= R && jj < R + TYT) Y[jj] = q[sc][jj - R];
        else Y[jj] = ldv(su + sc * C::U_STAGE + (C::SWZ ? uzc(jj) : yo(jj)));
        if (SEAM && yzero_warp && jj == yzero) Y[jj] = V{};
      }
      // x neighbours: KX vectors on each side of the centre vector
      V XL[TYT][KX], XR[TYT][KX];
#pragma unroll
      for (int r = 0; r < TYT; ++r)
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          if (C::SWZ) {
            // chunks kc -+ 1 of my own row: the centre chunk's swizzled index xor 1 ... via the packed field
            const int rr = ly * TYT + R + r;
            const int cc = (int)((zsw >> (3 * ((R + r) & 7))) & 7u);        // kc ^ (rr & 7)
            XL[r][k] = ldv(su + sc * C::U_STAGE + rr * C::SW + ((cc ^ (kcv ^ (kcv - (KX - k)))) * NV));
            XR[r][k] = ldv(su + sc * C::U_STAGE + rr * C::SW + ((cc ^ (kcv ^ (kcv + k + 1))) * NV));
          } else {
            XL[r][k] = ldv(S + r * C::SW - (KX - k) * NV);
            XR[r][k] = ldv(S + r * C::SW + (k + 1) * NV);
          }
          if (SEAM && xl_zero) XL[r][k] = V{};
          if (SEAM && xr_zero) XR[r][k] = V{};
        }
      T X[TYT][(2 * KX + 1) * NV];           // x-4.. of my points, centre at XC
#pragma unroll
      for (int r = 0; r < TYT; ++r)
#pragma unroll
        for (int e = 0; e < NV; ++e) {
#pragma unroll
          for (int k = 0; k < KX; ++k) {
            X[r][k * NV + e] = vget(XL[r][k], e);
            X[r][XC + NV + k * NV + e] = vget(XR[r][k], e);
          }
          X[r][XC + e] = vget(Y[R + r], e);
        }
      T L[TYT][NV];
      // fp32: the 25-point sum on packed pairs of x-points (FMUL2/FADD2/FFMA2,
      // bitwise the scalar chain below element by element, half the issue slots)
      constexpr bool PK = sizeof(T) == 4 && W25_PACKED &&
                          (INN || (W25_PACK_WALLY && MODE == MODE_WALLY) || (W25_PACK_WALLX && MODE == MODE_WALLX));
      if (PK && MODE != MODE_NULL) {
        f2_t L2[TYT][2];
        auto pr = [&](const V& v, int h) -> f2_t {
          return f2_pack((float)vget(v, 2 * h), (float)vget(v, 2 * h + 1));
        };
        // centre and x terms scalar (the x-neighbour pairs of odd m straddle
        // register pairs: repacking them would cost what packing saves), then
        // y and z terms on pairs -- the same per-element chain order as below
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          T Lx[NV];
#pragma unroll
          for (int c = 0; c < NV; ++c) {
            Lx[c] = mul_rn(K.c0, vget(Y[R + r], c));
#pragma unroll
            for (int m = 1; m <= R; ++m) Lx[c] = fma_rn(K.cx[m - 1], add_rn(X[r][XC + c + m], X[r][XC + c - m]), Lx[c]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) L2[r][h] = f2_pack((float)Lx[2 * h], (float)Lx[2 * h + 1]);
        }
#pragma unroll
        for (int m = 1; m <= R; ++m)
#pragma unroll
          for (int r = 0; r < TYT; ++r)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              L2[r][h] = f2_fma(f2_bcast((float)K.cy[m - 1]), f2_add(pr(Y[R + r + m], h), pr(Y[R + r - m], h)),
                                L2[r][h]);
#pragma unroll
        for (int m = 1; m <= R; ++m)
#pragma unroll
          for (int r = 0; r < TYT; ++r)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              L2[r][h] = f2_fma(f2_bcast((float)K.cz[m - 1]),
                                f2_add(pr(q[(s + 4 + m) % 9][r], h), pr(q[(s + 4 - m + 9) % 9][r], h)), L2[r][h]);
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float lo, hi;
            f2_unpack(L2[r][h], lo, hi);
            L[r][2 * h] = (T)lo;
            L[r][2 * h + 1] = (T)hi;
          }
      } else {
#pragma unroll
      for (int r = 0; r < TYT; ++r)
#pragma unroll
        for (int c = 0; c < NV; ++c) L[r][c] = mul_rn(K.c0, vget(Y[R + r], c));
      if (MODE != MODE_NULL) {
#pragma unroll
      for (int m = 1; m <= R; ++m)
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < NV; ++c)
            L[r][c] = fma_rn(K.cx[m - 1], add_rn(X[r][XC + c + m], X[r][XC + c - m]), L[r][c]);
#pragma unroll
      for (int m = 1; m <= R; ++m)
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < NV; ++c)
            L[r][c] = fma_rn(K.cy[m - 1], add_rn(vget(Y[R + r + m], c), vget(Y[R + r - m], c)), L[r][c]);
#pragma unroll
      for (int m = 1; m <= R; ++m)
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < NV; ++c)
            L[r][c] = fma_rn(K.cz[m - 1],
                             add_rn(vget(q[(s + 4 + m) % 9][r], c), vget(q[(s + 4 - m + 9) % 9][r], c)),
                             L[r][c]);
      }
      }

      // 3. u^{n-1}, vdt2 of plane z
      const int po_ = 9 * j + s;             // plane index in the chunk
      const int sp = po_ % C::SPN;
      mbar_wait(&full_p[sp], (po_ / C::SPN) & 1);
      V upv[TYT], vv[TYT];
#pragma unroll
      for (int r = 0; r < TYT; ++r) {
        upv[r] = ldv(sup + sp * C::P_STAGE + po + r * CW);
        vv[r] = ldv(sv + sp * C::P_STAGE + po + r * CW);
      }
      float ecur[ES ? TYT : 1][ES ? NV : 1], ecur_xm[ES ? TYT : 1][ES ? NV : 1], ecur_xp[ES ? TYT : 1][ES ? NV : 1];
      float ecur_ym[ES ? TYT : 1][ES ? NV : 1], ecur_yp[ES ? TYT : 1][ES ? NV : 1], enext[ES ? TYT : 1][ES ? NV : 1];
      if (ES) {
        // my eta box cell: row ly*TYT + r + 1, column NV*lx + 4 (+c); phantom
        // lanes clamp to the box (their results are masked)
        const int ec = min(NV * lx, CW - NV) + 4;
        const float* E0 = se + sp * C::E_STAGE;
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          const float* row = E0 + (ly * TYT + r + 1) * C::EW + ec;
#pragma unroll
          for (int c = 0; c < NV; ++c) {
            ecur[r][c] = row[c];
            ecur_xm[r][c] = row[c - 1];
            ecur_xp[r][c] = row[c + 1];
            ecur_ym[r][c] = row[c - C::EW];
            ecur_yp[r][c] = row[c + C::EW];
          }
        }
        // z + 1: the next plane's stage (issued ahead by the producer), or
        // past the chunk end from global memory (0 outside the domain)
        if (z + 1 < ze) {
          const int pn = po_ + 1, spn = pn % C::SPN;
          mbar_wait(&full_p[spn], (pn / C::SPN) & 1);
          const float* E1 = se + spn * C::E_STAGE;
#pragma unroll
          for (int r = 0; r < TYT; ++r)
#pragma unroll
            for (int c = 0; c < NV; ++c) enext[r][c] = E1[(ly * TYT + r + 1) * C::EW + ec + c];
        } else {
#pragma unroll
          for (int r = 0; r < TYT; ++r)
#pragma unroll
            for (int c = 0; c < NV; ++c) {
              const int x = gx + c, y = gy + r;
              enext[r][c] = (z + 1 < P.nzl && x < P.nx && y < P.ny)
                                ? __ldg(P.eta + ((int64_t)(z + 1) * P.ny + y) * P.pitch + x) : 0.f;
            }
        }
      }
      // all smem reads of plane z done: release its stages to the producer
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_u[sc]);
        if (CL > 1 && crank < CL - 1) mbar_arrive_remote(rem_empty + 8 * sc);
        mbar_arrive(&empty_p[sp]);
      }

      // 4. update (one uniform branch per plane) and store
      const int kg = z + P.zoff;
      V res[TYT];
      if (MODE == MODE_NULL) {
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          T o[NV];
#pragma unroll
          for (int c = 0; c < NV; ++c) o[c] = vget(upv[r], c) + vget(vv[r], c) + (c == 0 ? L[r][0] : T(0));
          res[r] = vmake<T>(o);
        }
      } else if (INN || (MODE == MODE_FUSED && !warp_xy_pml)) {
        if (kg >= P.w && kg < P.nzg - P.w) {
#pragma unroll
          for (int r = 0; r < TYT; ++r) {
            T o[NV];
            if (PK) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                float lo, hi;
                f2_unpack(f2_upd_inner(f2_pack((float)L[r][2 * h], (float)L[r][2 * h + 1]),
                                       f2_pack((float)vget(Y[R + r], 2 * h), (float)vget(Y[R + r], 2 * h + 1)),
                                       f2_pack((float)vget(upv[r], 2 * h), (float)vget(upv[r], 2 * h + 1)),
                                       f2_pack((float)vget(vv[r], 2 * h), (float)vget(vv[r], 2 * h + 1))),
                          lo, hi);
                o[2 * h] = (T)lo;
                o[2 * h + 1] = (T)hi;
              }
            } else {
#pragma unroll
              for (int c = 0; c < NV; ++c) o[c] = upd_inner(L[r][c], vget(Y[R + r], c), vget(upv[r], c), vget(vv[r], c));
            }
            res[r] = vmake<T>(o);
          }
        } else {
          const int dz = dist1(kg, P.nzg, P.w);
          CapCT<T> cc;
          cc.ex = stab[dz];
          cc.ezp = stab[dist1(kg + 1, P.nzg, P.w)];
          cc.ezm = stab[dist1(kg - 1, P.nzg, P.w)];
          cc.A = stab[TABN + dz];
          cc.B = stab[2 * TABN + dz];
          cc.rB = stab[3 * TABN + dz];
#pragma unroll
          for (int r = 0; r < TYT; ++r) {
            T xpa[NV], xma[NV];
#pragma unroll
            for (int c = 0; c < NV; ++c) { xpa[c] = X[r][XC + c + 1]; xma[c] = X[r][XC + c - 1]; }
            res[r] = cap_update<T>(vmake<T>(L[r]), Y[R + r], upv[r], vv[r], vmake<T>(xpa), vmake<T>(xma),
                                   Y[R + r + 1], Y[R + r - 1], q[(s + 5) % 9][r], q[(s + 3) % 9][r], cc, K.i2h[0],
                                   K.i2h[1], K.i2h[2], P.fastdiv != 0);
          }
        }
      } else if (MODE == MODE_WALL_ETA) {
        // stored (user-supplied) eta, staged by TMA in the u_prev/vdt2 ring
        // (box (CW+8) x (TY+2) per plane): x/y neighbours and the point from
        // plane z's stage, z+1 from the next stage (loaded ahead), z-1 carried
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          T xpa[NV], xma[NV];
#pragma unroll
          for (int c = 0; c < NV; ++c) { xpa[c] = X[r][XC + c + 1]; xma[c] = X[r][XC + c - 1]; }
          res[r] = pml_row_eta_s<T>(vmake<T>(L[r]), Y[R + r], upv[r], vv[r], vmake<T>(xpa), vmake<T>(xma),
                                    Y[R + r + 1], Y[R + r - 1], q[(s + 5) % 9][r], q[(s + 3) % 9][r], gx, gy + r, z,
                                    PG, ecur[r], ecur_xm[r], ecur_xp[r], ecur_ym[r], ecur_yp[r], eprev[r], enext[r],
                                    P.dt);
#pragma unroll
          for (int c = 0; c < NV; ++c) eprev[r][c] = ecur[r][c];
        }
      } else if (wallw && wkind != 0 && kg > P.w && kg < P.nzg - P.w - 1) {
        // wall, z-interior plane, pure y-wall rows (g = gy) or pure x-wall
        // columns (g = gx); the other two grad terms are +-0 exactly (dropped)
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          T o[NV];
          T num[NV], Bd[NV], rBd[NV];
          if (MODE == MODE_WALLY || (MODE != MODE_WALLX && MODE != MODE_SEAM && wkind == 1)) {
            const int ri = ly * TYT + r;
            const T cg = s_wr[ri], Aw = s_wr[TY + ri], Bw = s_wr[2 * TY + ri], rBw = s_wr[3 * TY + ri];
#pragma unroll
            for (int c = 0; c < NV; ++c) {
              const T gya = mul_rn(cg, mul_rn(sub_rn(vget(Y[R + r + 1], c), vget(Y[R + r - 1], c)), K.i2h[1]));
              num[c] = pml_num(L[r][c], gya, X[r][XC + c], vget(upv[r], c), vget(vv[r], c), Aw);
              Bd[c] = Bw;
              rBd[c] = rBw;
            }
          } else {
            const V cgv = ldv(s_wc + wci), Av = ldv(s_wc + CW + wci), Bv = ldv(s_wc + 2 * CW + wci);
            const V rBv = ldv(s_wc + 3 * CW + wci);
#pragma unroll
            for (int c = 0; c < NV; ++c) {
              const T gxa = mul_rn(vget(cgv, c), mul_rn(sub_rn(X[r][XC + c + 1], X[r][XC + c - 1]), K.i2h[0]));
              num[c] = pml_num(L[r][c], gxa, X[r][XC + c], vget(upv[r], c), vget(vv[r], c), vget(Av, c));
              Bd[c] = vget(Bv, c);
              rBd[c] = vget(rBv, c);
            }
          }
          div_table_row<T, NV>(num, Bd, rBd, P.fastdiv != 0, o);
          res[r] = vmake<T>(o);
        }
      } else {
        // wall plane in / next to a z cap, or a fused-mode warp touching the x/y
        // PML: full 7-point eta star per point (d = 0 points take the inner formula)
#pragma unroll
        for (int r = 0; r < TYT; ++r) {
          T xpa[NV], xma[NV];
#pragma unroll
          for (int c = 0; c < NV; ++c) { xpa[c] = X[r][XC + c + 1]; xma[c] = X[r][XC + c - 1]; }
          res[r] = pml_row_call<T>(vmake<T>(L[r]), Y[R + r], upv[r], vv[r], vmake<T>(xpa), vmake<T>(xma),
                                   Y[R + r + 1], Y[R + r - 1], q[(s + 5) % 9][r], q[(s + 3) % 9][r], px, py + r,
                                   kg, PG, stab, P.fastdiv != 0);
        }
      }
      if (PAIR && src_r >= 0 && z == P.src_k) {
        const unsigned long long n = *P.dstep + (unsigned long long)(role - 1);
        if (n < (unsigned long long)P.ninc) {
#pragma unroll
          for (int r = 0; r < TYT; ++r)
            if (r == src_r) {
              T o[NV];
#pragma unroll
              for (int c = 0; c < NV; ++c) o[c] = vget(res[r], c);
              o[src_c] = add_rn(o[src_c], static_cast<const T*>(P.inc)[n]);
              res[r] = vmake<T>(o);
            }
        }
      }
      if (full) {
        if ((PAIR && role == 1) || P.st_keep) {
          // u^{n+1} is re-read from L2 by the step-2 blocks: normal (not evict-first) stores
#pragma unroll
          for (int r = 0; r < TYT; ++r) *reinterpret_cast<V*>(optr + r * P.pitch) = res[r];
        } else {
#pragma unroll
          for (int r = 0; r < TYT; ++r) st_cs_v(optr + r * P.pitch, res[r]);
        }
      } else {
#pragma unroll
        for (int r = 0; r < TYT; ++r)
#pragma unroll
          for (int c = 0; c < NV; ++c)
            if (mask & (1u << (r * NV + c))) optr[r * P.pitch + c] = vget(res[r], c);
      }
      // fused halo exchange: edge planes also go straight into the neighbour's
      // ghost planes over the peer mapping (plane-uniform branches).  The two
      // targets are independent: on a slab of fewer than 2R planes a plane can
      // be an edge plane of both faces and must reach both neighbours.
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        T* rbase = nullptr;
        if (side == 0 && z < R && P.rlo) rbase = static_cast<T*>(P.rlo) + (int64_t)z * P.plane;
        if (side == 1 && z >= P.nzl - R && P.rhi) rbase = static_cast<T*>(P.rhi) + (int64_t)(z - (P.nzl - R)) * P.plane;
        if (rbase) {
          T* rp = rbase + (int64_t)gy * P.pitch + gx + sadj;
          if (full) {
#pragma unroll
            for (int r = 0; r < TYT; ++r) *reinterpret_cast<V*>(rp + r * P.pitch) = res[r];
          } else {
#pragma unroll
            for (int r = 0; r < TYT; ++r)
#pragma unroll
              for (int c = 0; c < NV; ++c)
                if (mask & (1u << (r * NV + c))) rp[r * P.pitch + c] = vget(res[r], c);
          }
        }
      }
      if (PAIR && role == 1) {
        // publish planes ..z (every pair_pk planes and at the end) once every
        // consumer warp has stored its part: each warp arrives on the
        // publication's slot (acq_rel, CTA scope); the last one adds the planes
        // to the tile's counter with a gpu-scope release, which (cumulative)
        // covers all the warps' stores.  Publications complete in order, so the
        // counter = the number of finished planes.  (One gpu-scope release per
        // plane costs ~1 us of store drain each: amortised over pair_pk planes.)
        const int zr = z - zs;
        if (zr % P.pair_pk == P.pair_pk - 1 || z == ze - 1) {
          __syncwarp();
          if (lane == 0 && !(P.pair_dbg & 2)) {
            const unsigned e = (unsigned)(zr / P.pair_pk);
            const unsigned old = atom_acqrel_cta_shared_add(&s_arr[e & 15], 1u);
            if (old == ((e >> 4) + 1) * (unsigned)C::NWC - 1u)
              red_release_gpu_add(P.prog + (int64_t)zc * G.ntx * G.nty + tyi * G.ntx + txi,
                                  (unsigned)(zr - (int)e * P.pair_pk + 1));
          }
        }
      }
      optr += P.plane;
      // embedded walls: the interior's progress paces the wall warps' claims
      if (EW && tid == 0)
        *reinterpret_cast<volatile int*>(smem_raw + C::EW_OFF + (SU * EW_US + 2 * EW_SPN * EW_PS + EW_COEF) * 4 +
                                         2 * (SU + EW_SPN) * 8) = z + 1 - zs;
    }
  }
  if (CL > 1) cluster_sync_all();           // the next CTA's consumers may still arrive on our barriers
}

template <int TX, int CW, int TY, int TYT, int MODE, int MINB, int RA = 0, typename T = float, int PAIR = 0,
          int CL = 1>
__global__ void __maxnreg__((StreamCfg<TX, CW, TY, TYT, MINB, RA, T>::MAXR))
k_stream(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_up,
         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ StreamParams P) {
  stream_body<TX, CW, TY, TYT, MODE, MINB, RA, T, PAIR, CL>(tm_u, tm_up, tm_v, P, blockIdx.x);
}

// ---------------------------------------------------------------------------
// k_mix: the interior launch and the x-wall launch as ONE grid.
// Work units of both are interleaved chunk by chunk: z-chunk c holds the
// interior's tiles (tile-row order) with the x-wall tiles of the same rows
// slotted in next to them, so a wall CTA streams its 64-B row pieces while the
// interior CTAs of the same rows and planes open the same DRAM pages and read
// the same halo columns through L2.  Every CTA is uniformly interior or wall
// (no per-warp paths); both bodies are the unchanged k_stream bodies, which
// need the same block size and register cap (checked on the host).
struct MixParams {
  StreamParams pi, pw;          // interior / x-wall launch parameters (same cz, same z range)
  const int* seq;               // per chunk position: >= 0 interior tile, < 0 -(1 + wall tile)
  int per_chunk;                // interior tiles + wall tiles per z-chunk
  int ni;                       // interior tiles per z-chunk
};

template <int TXI, int TYI, int TXW, int CWW, int TYW, int RA>
__global__ void __maxnreg__((StreamCfg<TXI, TXI, TYI, 1, 1, RA, float>::MAXR))
k_mix(const __grid_constant__ CUtensorMap ti_u, const __grid_constant__ CUtensorMap ti_up,
      const __grid_constant__ CUtensorMap ti_v, const __grid_constant__ CUtensorMap tw_u,
      const __grid_constant__ CUtensorMap tw_up, const __grid_constant__ CUtensorMap tw_v,
      const __grid_constant__ MixParams M) {
  static_assert(StreamCfg<TXI, TXI, TYI, 1, 1, RA, float>::NT == StreamCfg<TXW, CWW, TYW, 1, 1, RA, float>::NT,
                "interior and wall bodies need the same block size");
  const int c = blockIdx.x / M.per_chunk;
  const int q = M.seq[blockIdx.x - c * M.per_chunk];
  if (q >= 0) {
    stream_body<TXI, TXI, TYI, 1, MODE_INNER, 1, RA, float, 0>(ti_u, ti_up, ti_v, M.pi, c * M.ni + q);
  } else {
    // wall tile s of chunk c: region s / ncol, tile s % ncol (regions are
    // region-major in the wall launch's own numbering)
    const int s = -q - 1;
    const Region& g0 = M.pw.reg[0];
    const int ncol = g0.ntx * g0.nty;
    const int r = s / ncol;
    stream_body<TXW, CWW, TYW, 1, MODE_WALLX, 1, RA, float, 0>(tw_u, tw_up, tw_v, M.pw,
                                                             M.pw.reg[r].blk0 + c * ncol + (s - r * ncol));
  }
}

}  // namespace w25
