// wave.cu -- host side of the C ABI declared in include/wave.h.
//
// Owns: validation, fp64->fp32 constant tables, TMA descriptor encoding,
// region/tile/chunk planning, launch of the streaming kernels (interior column
// + x walls + y walls, forked on two streams and joined), the source kernel,
// CUDA-graph capture of 2-step pairs, and the split-step calls used by the
// z-slab multi-GPU driver.  No torch types cross this boundary.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>   // PFN_cuTensorMapEncodeTiled

#include "../../include/wave.h"
#include "aux_kernels.cuh"
#include "stream.cuh"
#include "tb2.cuh"
#include "paper_shapes.cuh"

using namespace w25;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static wave_status fail(wave_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(WAVE_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define CKST(expr)                          \
  do {                                      \
    wave_status s_ = (expr);                \
    if (s_ != WAVE_OK) return s_;           \
  } while (0)

// ---------------------------------------------------------------------------
// kernel configurations (tile shapes)
// ---------------------------------------------------------------------------
struct KInfo {
  void* fn;
  int tx, cw, ty, nt;      // TMA box width, computed width, tile height, threads
  size_t (*smem)(int w);
  const char* name;
  int cl = 1;              // thread-block cluster size (y-stacked tiles, multicast u halves)
  bool swz = false;        // u boxes loaded with the TMA 128-B swizzle (StreamCfg::SWZ)
};

template <int TX, int CW, int TY, int TYT, int MODE, int MINB = 2, int RA = 0, typename T = float, int PAIR = 0,
          int CL = 1>
static KInfo kinfo(const char* name) {
  using C = StreamCfg<TX, CW, TY, TYT, MINB, RA, T, MODE == MODE_WALL_ETA, MODE == MODE_INNER_EW ? EW_BYTES : 0>;
  // tx = width of the u TMA box minus its halo (the half width for split boxes)
  return KInfo{(void*)k_stream<TX, CW, TY, TYT, MODE, MINB, RA, T, PAIR, CL>, C::HW, CW, TY, C::NT, &C::smem_bytes,
               name, CL, C::SWZ};
}

// interior-kernel variants (WAVE25_INNER_TILE selects one; default first)
static const KInfo* inner_variants(int* n) {
  static const KInfo v[] = {
      kinfo<248, 248, 8, 1, MODE_INNER, 1, 112>("248x8x1r"),
      kinfo<248, 248, 8, 1, MODE_INNER, 1, 112, float, 0, 2>("248x8x1rc2"),
      kinfo<248, 248, 8, 1, MODE_INNER, 1, 112, float, 0, 4>("248x8x1rc4"),
      kinfo<128, 128, 8, 1, MODE_INNER>("128x8x1"),
      kinfo<128, 128, 16, 1, MODE_INNER, 1>("128x16x1"),
      kinfo<64, 64, 16, 1, MODE_INNER>("64x16x1"),
      kinfo<128, 128, 8, 2, MODE_INNER, 1>("128x8x2"),
      kinfo<128, 128, 8, 1, MODE_NULL>("null128x8x1"),      // memory-pattern probe (wrong results!)
      kinfo<128, 128, 8, 1, MODE_FUSED>("fused128x8x1"),
      kinfo<128, 128, 16, 1, MODE_NULL, 1>("null128x16x1"),
      kinfo<248, 248, 8, 1, MODE_INNER, 1>("248x8x1"),
      kinfo<240, 240, 8, 1, MODE_INNER, 1, 112>("240x8x1r"),
      kinfo<256, 256, 8, 1, MODE_INNER, 1, 112>("256x8x1r"),
      kinfo<248, 248, 8, 2, MODE_INNER, 1>("248x8x2"),
      // two rows per thread (y-neighbour LDS per row 8 -> 4: the interior is
      // close to shared-memory-bound, ncu l1tex 78 %): 8 consumer warps at 232
      // registers + the producer warpgroup at 24
      kinfo<248, 248, 8, 2, MODE_INNER, 1, 232>("248x8x2r"),
      kinfo<248, 248, 8, 1, MODE_INNER, 1, 104>("248x8x1r104"),   // consumers at 104 registers (A/B)
      // two CTAs per SM (each a producer warpgroup at 24 + 8 consumer warps at 104 registers)
      kinfo<128, 128, 8, 1, MODE_INNER, 2, 104>("128x8x1r2"),
      kinfo<128, 124, 8, 1, MODE_INNER, 2, 104>("c124x8x1r2"),
      kinfo<248, 248, 4, 1, MODE_INNER, 1>("248x4x1"),
      kinfo<248, 248, 8, 2, MODE_NULL, 1>("null248x8x2"),
      kinfo<224, 224, 4, 1, MODE_INNER, 1>("224x4x1"),
      kinfo<224, 224, 8, 1, MODE_INNER, 1>("224x8x1"),
      kinfo<224, 224, 4, 1, MODE_NULL, 1>("null224x4x1"),
      kinfo<224, 224, 8, 1, MODE_NULL, 1>("null224x8x1"),
  };
  *n = (int)(sizeof v / sizeof v[0]);
  return v;
}

// x walls: 16 computed columns per tile; 24 + 8 = 32-float (128-B) u boxes
static const KInfo* wallx_variants(int* n) {
  static const KInfo v[] = {
      kinfo<24, 16, 128, 1, MODE_WALLX, 1, 112>("x24c16x128x1r"),
      kinfo<24, 16, 128, 1, MODE_WALL, 1, 112>("x24c16x128x1rg"),     // generic wall body (A/B)
      kinfo<24, 16, 64, 1, MODE_WALLX, 2, 104>("x24c16x64x1r2"),      // two CTAs per SM
      kinfo<24, 16, 32, 1, MODE_WALL>("x24c16x32x1"),
      kinfo<28, 16, 32, 1, MODE_WALL>("x28c16x32x1"),
      kinfo<24, 16, 64, 1, MODE_WALL, 1, 232>("x24c16x64x1r"),
      kinfo<40, 32, 64, 1, MODE_WALL, 1, 112>("x40c32x64x1r"),
      kinfo<28, 16, 64, 1, MODE_WALL, 1>("x28c16x64x1"),
      kinfo<28, 16, 32, 1, MODE_WALL, 3>("x28c16x32x1m3"),
      kinfo<24, 16, 32, 1, MODE_WALL, 3>("x24c16x32x1m3"),
      kinfo<24, 16, 32, 1, MODE_WALL, 4>("x24c16x32x1m4"),
      kinfo<32, 16, 32, 1, MODE_WALL>("x32c16x32x1"),
      kinfo<24, 16, 64, 1, MODE_WALL, 1>("x24c16x64x1"),
      kinfo<32, 16, 64, 1, MODE_WALL, 1>("x32c16x64x1"),
      kinfo<32, 32, 32, 1, MODE_WALL>("x32c32x32x1"),
  };
  *n = (int)(sizeof v / sizeof v[0]);
  return v;
}

static const KInfo* wally_variants(int* n) {
  static const KInfo v[] = {
      kinfo<128, 128, 16, 1, MODE_WALLY, 1, 112>("y128x16x1r"),
      kinfo<128, 128, 16, 1, MODE_WALL, 1, 112>("y128x16x1rg"),      // generic wall body (A/B)
      kinfo<128, 128, 8, 1, MODE_WALLY, 2, 104>("y128x8x1r2"),        // two CTAs per SM
      kinfo<248, 248, 8, 1, MODE_WALLY, 1, 112>("y248x8x1ry"),         // the interior's tile shape
      kinfo<64, 64, 8, 1, MODE_WALL, 3>("y64x8x1m3"),
      kinfo<248, 248, 8, 1, MODE_WALL, 1, 112>("y248x8x1r"),
      kinfo<64, 64, 16, 1, MODE_WALL, 2>("y64x16x1m2"),
      kinfo<128, 128, 8, 1, MODE_WALL, 3>("y128x8x1m3"),
      kinfo<128, 128, 8, 1, MODE_WALL, 1>("y128x8x1"),
      kinfo<128, 128, 8, 1, MODE_WALL, 2>("y128x8x1m2"),
      kinfo<128, 128, 16, 1, MODE_WALL, 1>("y128x16x1"),
  };
  *n = (int)(sizeof v / sizeof v[0]);
  return v;
}

static KInfo pick(const KInfo* v, int n, const char* env) {
  const char* e = getenv(env);
  if (e)
    for (int i = 0; i < n; ++i)
      if (!strcmp(e, v[i].name)) return v[i];
  return v[0];
}

// KI_WALLX_E / KI_WALLY_E: the wall kernels of the stored-eta mode
// KI_PAIR: the two-step-through-L2 interior kernel
// KI_SEAM: both x walls as seams (MODE_SEAM)
// KI_EW: the interior kernel with embedded wall warps (MODE_INNER_EW)
// KI_EWALL: not launched -- the TMA maps (16 x 8 boxes) of KI_EW's wall warps
enum { KI_INNER = 0, KI_WALLX = 1, KI_WALLY = 2, KI_FUSED = 3, KI_WALLX_E = 4, KI_WALLY_E = 5, KI_PAIR = 6,
       KI_SEAM = 7, KI_EW = 8, KI_EWALL = 9, KI_N = 10 };
static bool is_wall(int ki) {
  return ki == KI_WALLX || ki == KI_WALLY || ki == KI_WALLX_E || ki == KI_WALLY_E || ki == KI_SEAM;
}

static KInfo g_k[2][KI_N];   // [precision: 0 fp32, 1 fp64][kernel kind]
// the two bodies k_mix instantiates: the default interior and x-wall kernels
static KInfo mix_inner() { return kinfo<248, 248, 8, 1, MODE_INNER, 1, 112>("248x8x1r"); }
static KInfo mix_wallx() { return kinfo<24, 16, 128, 1, MODE_WALLX, 1, 112>("x24c16x128x1r"); }
static void* mix_fn() { return (void*)k_mix<248, 8, 24, 16, 128, 112>; }
static void init_kernels() {
  static bool done = false;
  if (done) return;
  int n = 0;
  const KInfo* v = inner_variants(&n);
  g_k[0][KI_INNER] = pick(v, n, "WAVE25_INNER_TILE");
  v = wallx_variants(&n);
  g_k[0][KI_WALLX] = pick(v, n, "WAVE25_WALLX_TILE");
  v = wally_variants(&n);
  g_k[0][KI_WALLY] = pick(v, n, "WAVE25_WALLY_TILE");
  static const KInfo fv[] = {kinfo<256, 256, 8, 1, MODE_FUSED, 1, 112>("fused256x8x1r"),
                             kinfo<128, 128, 8, 1, MODE_FUSED>("fused128x8x1")};
  g_k[0][KI_FUSED] = pick(fv, 2, "WAVE25_FUSED_TILE");
  // fp64: 16-B lanes hold 2 doubles; 124 = 992 / 8 columns,
  // u box 132 doubles; same ring / warpgroup structure as the fp32 kernels
  g_k[1][KI_INNER] = kinfo<124, 124, 8, 1, MODE_INNER, 1, 112, double>("d124x8x1r");
  {
    static const KInfo dx[] = {kinfo<24, 16, 64, 1, MODE_WALLX, 1, 112, double>("dx24c16x64x1r"),
                               kinfo<24, 16, 32, 1, MODE_WALL, 1, 0, double>("dx24c16x32x1"),
                               kinfo<24, 16, 32, 1, MODE_WALLX, 1, 168, double>("dx24c16x32x1r")};
    static const KInfo dy[] = {kinfo<64, 64, 16, 1, MODE_WALLY, 1, 112, double>("dy64x16x1r"),
                               kinfo<32, 32, 8, 1, MODE_WALL, 3, 0, double>("dy32x8x1m3")};
    g_k[1][KI_WALLX] = pick(dx, 3, "WAVE25_DWALLX_TILE");
    g_k[1][KI_WALLY] = pick(dy, 2, "WAVE25_DWALLY_TILE");
  }
  {
    // stored-eta walls: producer-warpgroup shapes (x walls
    // 16 x 64, y walls + caps 128 x 16; C3 serialized 0.355 -> 0.333 and
    // 0.413 -> 0.335 ms/step, profiles/eta_tiles_r02dd.txt), older shapes as A/B
    static const KInfo ex[] = {kinfo<24, 16, 64, 1, MODE_WALL_ETA, 1, 112>("ex24c16x64x1r"),
                               kinfo<24, 16, 32, 1, MODE_WALL_ETA, 2>("ex24c16x32x1")};
    static const KInfo ey[] = {kinfo<128, 128, 16, 1, MODE_WALL_ETA, 1, 112>("ey128x16x1r"),
                               kinfo<64, 64, 8, 1, MODE_WALL_ETA, 3>("ey64x8x1m3"),
                               kinfo<128, 128, 8, 1, MODE_WALL_ETA, 1, 112>("ey128x8x1r")};
    g_k[0][KI_WALLX_E] = pick(ex, 2, "WAVE25_EWALLX_TILE");
    g_k[0][KI_WALLY_E] = pick(ey, 3, "WAVE25_EWALLY_TILE");
  }
  g_k[1][KI_WALLX_E] = kinfo<24, 16, 32, 1, MODE_WALL_ETA, 1, 0, double>("edx24c16x32x1");
  g_k[1][KI_WALLY_E] = kinfo<32, 32, 8, 1, MODE_WALL_ETA, 3, 0, double>("edy32x8x1m3");
  g_k[0][KI_PAIR] = kinfo<248, 248, 8, 1, MODE_INNER, 1, 112, float, 1>("pair248x8x1r");
  g_k[1][KI_PAIR] = kinfo<124, 124, 8, 1, MODE_INNER, 1, 112, double, 1>("dpair124x8x1r");
  g_k[1][KI_FUSED] = kinfo<64, 64, 8, 1, MODE_FUSED, 2, 0, double>("dfused64x8x1");
  {
    static const KInfo sv[] = {kinfo<32, 32, 64, 1, MODE_SEAM, 1, 112>("seam32x64r"),
                               kinfo<32, 32, 32, 1, MODE_SEAM, 2>("seam32x32")};
    g_k[0][KI_SEAM] = pick(sv, 2, "WAVE25_SEAM_TILE");
  }
  g_k[1][KI_SEAM] = g_k[1][KI_WALLX];   // (fp32 only; fp64 plans never build seam launches)
  g_k[0][KI_EW] = kinfo<248, 248, 8, 1, MODE_INNER_EW, 1, EW_RC>("ew248x8x1r");
  {
    KInfo m = g_k[0][KI_EW];                 // (same function and smem size: the attribute loops stay consistent)
    m.tx = EW_CW; m.cw = EW_CW; m.ty = EW_TY; m.swz = false; m.name = "ewall16x8";
    g_k[0][KI_EWALL] = m;
  }
  g_k[1][KI_EW] = g_k[1][KI_EWALL] = g_k[1][KI_INNER];   // (fp32 only)
  done = true;
}
#define KTX(ki) (P->kt[ki].tx)
#define KCW(ki) (P->kt[ki].cw)
#define KTY(ki) (P->kt[ki].ty)
#define KCL(ki) (P->kt[ki].cl)

// the fp32 interior tile per geometry (unless WAVE25_INNER_TILE names one):
// the width among 248 / 240 (u boxes of 256 / 248 <= the TMA box limit)
// whose tiles cover the inner row with the fewest idle lanes, 248 on a tie
// (C3: 992 = 4 x 248; C2: 480 = 2 x 240 -- 1.6 % faster than 2 x 248 there)
static KInfo pick_inner(const wave_desc& d, int prec) {
  if (prec != 0 || getenv("WAVE25_INNER_TILE")) return g_k[prec][KI_INNER];
  const int64_t W = d.nx - 2 * (int64_t)d.pml_width;
  if (W <= 0) return g_k[0][KI_INNER];
  int n = 0;
  const KInfo* v = inner_variants(&n);
  const KInfo* best = &g_k[0][KI_INNER];
  int64_t bw = (W + best->cw - 1) / best->cw * best->cw;
  for (int i = 0; i < n; ++i)
    if (!strcmp(v[i].name, "240x8x1r")) {
      const int64_t c = (W + v[i].cw - 1) / v[i].cw * v[i].cw;
      if (c < bw) { best = &v[i]; bw = c; }
    }
  return *best;
}

static constexpr double W8[5] = {-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0};
static constexpr int MAX_W = W25_MAX_W;

struct Maps {
  CUtensorMap u[4];      // wavefield buffer b with halo box
  CUtensorMap up[4];     // wavefield buffer b, tile box
  CUtensorMap v;         // vdt2, tile box
};

// two-step temporal-blocking kernel (tb2.cuh) variants; WAVE25_T2_TILE selects
struct T2Info {
  void* fn;
  int tx, ty, nt;
  size_t (*smem)(int w);
  const char* name;
};
template <int TX, int TY>
static T2Info t2info(const char* name) {
  using C = T2Cfg<TX, TY>;
  return T2Info{(void*)k_tb2<TX, TY>, TX, TY, C::NT, &C::smem_bytes, name};
}
static T2Info pick_t2() {
  static const T2Info v[] = {t2info<56, 14>("56x14"), t2info<56, 16>("56x16"), t2info<56, 24>("56x24")};
  const char* e = getenv("WAVE25_T2_TILE");
  if (e)
    for (const T2Info& t : v)
      if (!strcmp(e, t.name)) return t;
  return v[0];
}

struct T2Maps {
  CUtensorMap u[4];      // u^n, box (TX+16, TY+16)
  CUtensorMap up[4];     // u^{n-1}, box (TX+8, TY+8)
  CUtensorMap v1;        // vdt2, box (TX+8, TY+8)
  CUtensorMap v2;        // vdt2, box (TX, TY)
};

struct Launch {          // one streaming-kernel launch
  int ki = 0;
  int nblk = 0;
  StreamParams p{};
};

struct wave_plan {
  wave_desc d{};
  wave_layout_info L{};
  int dev = 0, nsm = 148;
  int prec = 0;                      // 0: fp32, 1: fp64 (desc.precision)
  size_t esz = 4;                    // bytes per element
  Coef coef{};                       // fp32 constants (rounded once)
  CoefT<double> coefd{};             // fp64 constants (unrounded)
  std::vector<float> tab_h;          // [3][w+2] fp32
  std::vector<double> tab_hd;        // [3][w+2] fp64
  void* tab_d = nullptr;
  float* buf[4] = {nullptr, nullptr, nullptr, nullptr};   // element (0,0,-4) of each buffer (= base + origin)
  float* base[4] = {nullptr, nullptr, nullptr, nullptr};  // the caller's allocations (element type by prec)
  float* vdt2 = nullptr;                                   // element (0,0,0) of vdt2 (= vdt2_base + origin)
  float* vdt2_base = nullptr;
  bool bound = false, have_vel = false, aux = false;
  float* eta_buf = nullptr;          // stored eta, caller-owned, vdt2 layout (wave_plan_bind_eta)
  bool eta_on = false;               // wave_set_eta installed a field
  float dt = 0.f;
  int cur = 0, prv = 1;              // buf[cur] holds u^n, buf[prv] u^{n-1}
  int64_t step = 0;
  // source
  bool src_set = false, src_local = false;
  int64_t si = 0, sj = 0, sk = 0;
  std::vector<float> wavelet;
  void* inc_d = nullptr;
  float* wl_d = nullptr;
  int64_t ninc = 0;
  unsigned long long* dstep = nullptr;
  Stats* stats_d = nullptr;
  // launch plans
  KInfo kt[KI_N];                    // this plan's kernel per kind (g_k, the interior tile chosen per geometry)
  Maps maps[KI_N];
  int occ[KI_N] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
  bool fused = false;                // WAVE25_FUSED=1: one launch, per-warp paths (measured slower)
  int pf = 1;                        // L2 prefetch distance (WAVE25_PF), measured best
  int wall_pf = -1;                  // wall kernels' L2 prefetch distance (WAVE25_WALL_PF; -1 = pf)
  int prio_lo = 0, prio_hi = 0;      // stream priority range (launch attribute)
  bool wall_prio = true;             // WAVE25_WALL_PRIO=0 disables
  bool serial = false;               // WAVE25_SERIAL=1: walls and interior on one stream (diagnostic)
  bool xfuse = false;                // WAVE25_XFUSE=1: x walls computed inside the interior tiles
  int order = 0;                     // tile order (WAVE25_ORDER)
  int l2_persist_mb = 0;             // L2 set-aside for u (WAVE25_L2MB), 0 = off
  float l2_hit_ratio = 1.f;          // WAVE25_L2HR
  size_t max_window = 0;
  int upol = 0;                      // u L2 policy (WAVE25_UPOL)
  std::vector<Launch> launches[3];   // [0] all planes, [1] edges, [2] interior
  Maps* maps_g = nullptr;            // device copy of maps[] (WAVE25_GMAPS=1)
  bool gmaps = false;
  // streams / graphs
  cudaStream_t side = nullptr, cap = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t side2 = nullptr;      // y walls when side2_on (WAVE25_SIDE2)
  cudaEvent_t ev_join2 = nullptr;
  bool side2_on = false;            // set at plan creation (fp32: on)
  int wall_cz = 0;                   // WAVE25_WALL_CZ: wall chunk length (0 = auto)
  int xwall_extra = 0;               // WAVE25_XWALL_EXTRA: inner columns computed by the x-wall kernel
  bool xinter = true;                // WAVE25_XINTER=0: x-wall launch region-major instead of left/right interleaved
  bool fastdiv_on = true;            // WAVE25_FASTDIV=0: IEEE division in the PML updates (A/B)
  bool seam_on = false;              // WAVE25_SEAM=1: the x walls as seams (measured slower; A/B)
  bool fastdiv = false;              // table division verified bitwise for this plan (check_fastdiv)
  bool walls_last = false;           // WAVE25_WALLS_LAST: enqueue the wall kernels after the interior
  bool walls_alt = false;            // WAVE25_WALLS_ALT: walls last / first in the two steps of a graph
  bool wall_keep = false;            // WAVE25_WALL_STKEEP: wall u_next stores evict-normal
  int mix = 0;                       // WAVE25_MIX=1/2: interior + x walls as one grid (k_mix, §5i; measured slower)
  bool mix_ok = false;               // geometry / kernel choice supports k_mix (set by build_launches)
  int* mix_seq_d = nullptr;          // k_mix chunk sequence (device)
  MixParams mixp{};
  int mix_nblk = 0;
  cudaGraphExec_t gexec[16] = {};    // 2-step graphs keyed by (cur, prv)
  // two-step temporal blocking (WAVE_KERNEL_TB2)
  T2Info t2{};
  T2Maps t2maps{};
  bool t2_ok = false;                // plan geometry supports it (else single steps)
  int occ_t2 = 1;
  T2Params t2p{};
  int t2_nblk = 0;
  std::vector<Launch> wall_p1, wall_p2;  // walls: u^{n+1} on the (w+8)-frame, u^{n+2} on the (w+4)-frame
  cudaGraphExec_t gexec2[16] = {};   // 1-pair graphs keyed by (cur, prv)
  // two steps through L2 (WAVE_KERNEL_PAIR)
  bool pair_ok = false;
  Launch pair_launch;
  int* pair_groups_d = nullptr;
  int pair_dbg = 0;                  // WAVE25_PAIR_DBG timing probes (results invalid when set)
  int pair_pk = 16;                  // WAVE25_PAIR_PK: planes per step-1 progress publication
  int pair_cz = 256;                 // WAVE25_PAIR_CZ: z chunk of the pair kernel's blocks
  unsigned* prog_d = nullptr;
  int64_t prog_n = 0;
  cudaGraphExec_t gexecP[16] = {};
  // fused peer-store halo exchange
  bool have_peers = false;
  wave_peers peers{};
  unsigned long long* ddone = nullptr;     // [0] steps completed (flag protocol), [1] peer-wait error bits
  double peer_timeout_s = 300.0;           // k_peer_wait bound (WAVE25_PEER_TIMEOUT_S / wave_set_peer_timeout)
  bool remote = false;                     // enqueue with remote edge stores
  cudaGraphExec_t gexec_peer[2] = {nullptr, nullptr};
  // embedded wall warps (MODE_INNER_EW)
  bool ew_on = false;                      // WAVE25_EW=1
  int ew_cz = 0;                           // WAVE25_EW_CZ: wall unit length in planes (0 = auto)
  int ew_rem = -1;                         // WAVE25_EW_REM: claim while >= this many interior planes remain (-1 = cz)
  unsigned* ew_ctr = nullptr;              // [3 launch sets][2] tickets (self-resetting)
  int ew_pf = 8;                           // WAVE25_EW_PF: L2 prefetch distance of the wall loads
  unsigned long long* ew_dbg = nullptr;    // WAVE25_EW_DBG=1: wall-unit timing probe (6 counters)
};

// element-offset pointer into a buffer of the plan's precision
static inline float* eo(const wave_plan* P, const void* base, int64_t elems) {
  return reinterpret_cast<float*>(const_cast<char*>(static_cast<const char*>(base)) + elems * (int64_t)P->esz);
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static wave_status get_encoder() {
  if (g_encode) return WAVE_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    return fail(WAVE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return WAVE_OK;
}

// promotion of the centre-only (u_prev, vdt2) loads of kernel kind ki:
// WAVE25_WALL_L2PROMO for wall kernels whose rows are narrower than 128 B
static int centre_promo(const wave_plan* P, int ki, uint32_t cw) {
  static int v = [] {
    const char* e = getenv("WAVE25_WALL_L2PROMO");
    return e ? atoi(e) : -1;
  }();
  return (is_wall(ki) && cw * P->esz < 128) ? v : -1;
}

// L2 sector promotion of TMA loads (WAVE25_L2PROMO = 0 none, 1 64B, 2 128B, 3 256B);
// `v` >= 0 overrides it for one map
static CUtensorMapL2promotion l2_promotion(int v = -1) {
  static int dflt = [] {
    const char* e = getenv("WAVE25_L2PROMO");
    return e ? atoi(e) : 2;
  }();
  if (v < 0) v = dflt;
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 3: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
}

static wave_status encode3d(CUtensorMap* m, void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                            uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t b0, uint32_t b1,
                            bool f64 = false, int promo = -1, bool swz128 = false) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {pitch_bytes, plane_bytes};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base,
                        dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(promo),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(WAVE_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return WAVE_OK;
}

// ---------------------------------------------------------------------------
// validation and constants
// ---------------------------------------------------------------------------
static double courant_number(const wave_desc& d, double vmax, double dt) {
  // stability of leapfrog + Lap8: (V dt)^2 sum_a S/h_a^2 <= 4, S = max symbol
  // of the 1-D operator = -(w0 + 2 sum_m w_m cos(m pi)) = 6.5016...
  double S = -W8[0];
  for (int m = 1; m <= 4; ++m) S -= 2.0 * W8[m] * ((m & 1) ? -1.0 : 1.0);
  const double s = 1.0 / (d.hx * d.hx) + 1.0 / (d.hy * d.hy) + 1.0 / (d.hz * d.hz);
  return vmax * dt * std::sqrt(S * s) / 2.0;   // must be <= 1
}

static wave_status validate(const wave_desc* d) {
  if (!d) return fail(WAVE_ERR_CONFIG, "desc is NULL");
  if (d->nx < 1 || d->ny < 1 || d->nz < 1) return fail(WAVE_ERR_CONFIG, "extents must be >= 1");
  if (d->nx > (1 << 30) || d->ny > (1 << 30) || d->nz_global > (1 << 30))
    return fail(WAVE_ERR_CONFIG, "extent too large");
  if (d->nz_global < d->nz || d->z_offset < 0 || d->z_offset + d->nz > d->nz_global)
    return fail(WAVE_ERR_CONFIG, "slab [z_offset, z_offset+nz) must lie in [0, nz_global)");
  const int64_t w = d->pml_width;
  const int64_t mn = std::min(d->nx, std::min(d->ny, d->nz_global));
  if (w < 0 || 2 * w >= mn) return fail(WAVE_ERR_CONFIG, "need 0 <= 2w < min extent (w=%lld)", (long long)w);
  if (w > MAX_W) return fail(WAVE_ERR_CONFIG, "pml_width > %d", MAX_W);
  if (!(d->hx > 0 && d->hy > 0 && d->hz > 0) || !std::isfinite(d->hx) || !std::isfinite(d->hy) ||
      !std::isfinite(d->hz))
    return fail(WAVE_ERR_CONFIG, "spacing must be > 0");
  if (!(d->dt >= 0.f) || !std::isfinite(d->dt)) return fail(WAVE_ERR_CONFIG, "dt must be >= 0 (0 = auto)");
  if (!(d->eta_max >= 0) || !std::isfinite(d->eta_max)) return fail(WAVE_ERR_CONFIG, "eta_max must be >= 0");
  if (d->precision != WAVE_PREC_FP32 && d->precision != WAVE_PREC_FP64)
    return fail(WAVE_ERR_CONFIG, "unknown precision %d", d->precision);
  if (d->precision == WAVE_PREC_FP64 && d->kernel == WAVE_KERNEL_TB2)
    return fail(WAVE_ERR_CONFIG, "two-step blocking (TB2) is fp32 only");
  if (d->kernel == WAVE_KERNEL_PAIR && d->nz != d->nz_global)
    return fail(WAVE_ERR_CONFIG, "the two-step (PAIR) kernel needs a single-slab plan");
  if (d->kernel != WAVE_KERNEL_STREAM && d->kernel != WAVE_KERNEL_NAIVE && d->kernel != WAVE_KERNEL_TB2 &&
      d->kernel != WAVE_KERNEL_PAIR)
    return fail(WAVE_ERR_CONFIG, "unknown kernel %d", d->kernel);
  if (d->dt == 0.f && (d->nz != d->nz_global)) return fail(WAVE_ERR_CONFIG, "auto dt needs a single-slab plan");
  return WAVE_OK;
}

static void make_layout(const wave_desc& d, wave_layout_info* L) {
  L->pitch_x = (d.nx + 3) / 4 * 4;
  L->ghost_z = R;
  L->planes = d.nz + 2 * R;
  L->align_bytes = 128;
  L->elem_bytes = d.precision == WAVE_PREC_FP64 ? 8 : 4;
  // origin shift: when rows are whole 128-B lines, start every
  // row (w * elem_bytes) mod 128 bytes into a line, so that the first inner
  // column x = w is line-aligned: a 128-B line then holds either x-wall points
  // only (the right wall of row y and the left wall of row y+1) or inner points
  // only, and the interior and x-wall kernels (separate launches) never fetch
  // the same line from DRAM.  16-B granularity (TMA / vector alignment).
  L->origin = 0;
  static const bool no_origin = getenv("WAVE25_NO_ORIGIN") && atoi(getenv("WAVE25_NO_ORIGIN")) != 0;  // A/B only
  if ((L->pitch_x * L->elem_bytes) % 128 == 0 && !no_origin) {
    const int64_t sb = ((128 - (d.pml_width * L->elem_bytes) % 128) % 128) / 16 * 16;
    L->origin = sb / L->elem_bytes;
  }
  // seams (MODE_SEAM): fp32, w = 16 (one 128-B line = both walls), rows of
  // exactly nx elements; a seam view reads row -1 of the first plane and row ny
  // of the last one, so one pad row is kept before and after every buffer
  L->seam = d.precision == WAVE_PREC_FP32 && d.pml_width == 16 && L->pitch_x == d.nx && L->origin * 4 == 64 &&
            d.ny > 2 * d.pml_width && d.nx > 2 * d.pml_width;
  static const bool no_seam = getenv("WAVE25_NO_SEAM") && atoi(getenv("WAVE25_NO_SEAM")) != 0;   // A/B only
  if (no_seam) L->seam = 0;
  if (L->seam) L->origin += L->pitch_x;
  L->elems_u = L->origin + L->planes * d.ny * L->pitch_x + (L->seam ? L->pitch_x : 0);
  L->elems_vdt2 = L->origin + d.nz * d.ny * L->pitch_x + (L->seam ? L->pitch_x : 0);
}

// fp64 plans: every constant in fp64, never rounded to fp32
static void make_constants64(const wave_desc& d, float dt, CoefT<double>* k, std::vector<double>* tab) {
  const double ih2[3] = {1.0 / (d.hx * d.hx), 1.0 / (d.hy * d.hy), 1.0 / (d.hz * d.hz)};
  k->c0 = W8[0] * (ih2[0] + ih2[1] + ih2[2]);
  for (int m = 1; m <= 4; ++m) {
    k->cx[m - 1] = W8[m] * ih2[0];
    k->cy[m - 1] = W8[m] * ih2[1];
    k->cz[m - 1] = W8[m] * ih2[2];
  }
  for (int a = 0; a < 3; ++a) k->i2h[a] = 1.0 / (2.0 * (a == 0 ? d.hx : a == 1 ? d.hy : d.hz));
  const int w = d.pml_width, T = w + 2;
  tab->assign(4 * T, 0.0);
  for (int dd = 0; dd <= w; ++dd) {
    const double r = w > 0 ? (double)dd / (double)w : 0.0;
    const double eta = d.eta_max * r * r;
    (*tab)[dd] = eta;
    (*tab)[T + dd] = 1.0 - eta * (double)dt;
    (*tab)[2 * T + dd] = 1.0 + eta * (double)dt;
  }
  (*tab)[w + 1] = 0.0;
  (*tab)[T + w + 1] = 1.0;
  (*tab)[2 * T + w + 1] = 1.0;
  for (int i = 0; i < T; ++i) (*tab)[3 * T + i] = 1.0 / (*tab)[2 * T + i];   // unused (fp64 divides)
}

// RN(1/B) in fp32 exactly: the candidate from fp64 and its two neighbours,
// the one with the smallest |1 - r B| (exact in fp64: r B has 48 bits and
// lies within 2^-23 of 1).  1/B is never an fp32 midpoint (B > 1 is not a
// power of 2), so the minimum is unique.
static float recip_rn(float B) {
  const float c = (float)(1.0 / (double)B);
  float best = c;
  double be = 2.0;
  for (float r : {std::nextafter(c, 0.f), c, std::nextafter(c, 2.f)}) {
    const double e = std::fabs(1.0 - (double)r * (double)B);
    if (e < be) { be = e; best = r; }
  }
  return best;
}

// fp64 -> fp32 once (R8)
static void make_constants(const wave_desc& d, float dt, Coef* k, std::vector<float>* tab) {
  const double ih2[3] = {1.0 / (d.hx * d.hx), 1.0 / (d.hy * d.hy), 1.0 / (d.hz * d.hz)};
  k->c0 = (float)(W8[0] * (ih2[0] + ih2[1] + ih2[2]));
  for (int m = 1; m <= 4; ++m) {
    k->cx[m - 1] = (float)(W8[m] * ih2[0]);
    k->cy[m - 1] = (float)(W8[m] * ih2[1]);
    k->cz[m - 1] = (float)(W8[m] * ih2[2]);
  }
  k->i2h[0] = (float)(1.0 / (2.0 * d.hx));
  k->i2h[1] = (float)(1.0 / (2.0 * d.hy));
  k->i2h[2] = (float)(1.0 / (2.0 * d.hz));
  const int w = d.pml_width, T = w + 2;
  tab->assign(4 * T, 0.f);
  for (int dd = 0; dd <= w; ++dd) {
    const double r = w > 0 ? (double)dd / (double)w : 0.0;
    const double eta = d.eta_max * r * r;                 // eta_max (d/w)^2, R2
    (*tab)[dd] = (float)eta;
    (*tab)[T + dd] = (float)(1.0 - eta * (double)dt);
    (*tab)[2 * T + dd] = (float)(1.0 + eta * (double)dt);
  }
  (*tab)[w + 1] = 0.f;                                    // outside the domain (R4)
  (*tab)[T + w + 1] = 1.f;
  (*tab)[2 * T + w + 1] = 1.f;
  for (int i = 0; i < T; ++i) (*tab)[3 * T + i] = recip_rn((*tab)[2 * T + i]);   // RN(1/B_d), common.cuh div_table
}

// ---------------------------------------------------------------------------
// launch planning
// ---------------------------------------------------------------------------
static void* kernel_ptr(const wave_plan* P, int ki) { return P->kt[ki].fn; }
static int kernel_threads(const wave_plan* P, int ki) { return P->kt[ki].nt; }
static size_t kernel_smem(const wave_plan* P, int ki) { return P->kt[ki].smem(P->d.pml_width); }

// z-chunk length minimising (waves x (chunk + warm-up)) for ncol columns over nz planes
static int choose_cz(int64_t ncol, int nz, int resident, double warm = 4.0, int maxcz = 1 << 30) {
  int best = nz;
  double best_cost = 1e300;
  for (int k = 1; k <= 256; ++k) {
    const int cz = (nz + k - 1) / k;
    if (cz < 8 && k > 1) break;
    if (cz > maxcz && (nz + k) / (k + 1) >= 8) continue;
    const int64_t nch = (nz + cz - 1) / cz;
    const double waves = std::ceil((double)(ncol * nch) / std::max(1, resident));
    const double cost = waves * (cz + warm);   // warm-up planes cost ~ half a plane each
    if (cost < best_cost * 0.999) { best_cost = cost; best = cz; }
  }
  return best;
}

constexpr int W25_WALL_CZ_MAX = 40;    // longest fp32 wall z-chunk (measured, C3/C2)

struct ZRange { int z0, z1; };

// Build the region list of one launch kind over a set of z ranges.
static void add_regions(wave_plan* P, int ki, const std::vector<std::array<int, 4>>& xy,
                        const std::vector<ZRange>& zr, std::vector<Launch>* out);

// x walls as seams (MODE_SEAM): the layout reserved the pad rows (fp32, w = 16,
// rows of exactly nx), and no mode that shapes the x walls differently is on
static bool seam_active(const wave_plan* P) {
  return P->L.seam && P->prec == 0 && !P->eta_on && !P->fused && !P->xfuse && P->xwall_extra == 0 && P->seam_on &&
         P->d.kernel == WAVE_KERNEL_STREAM;
}

static const char* ablation_shape();

// embedded wall warps: fp32 default-path plans with PML walls only (any mode
// that shapes the interior or the walls differently keeps separate launches)
static bool ew_wanted(const wave_plan* P) {
  const int nx = (int)P->d.nx, ny = (int)P->d.ny, w = P->d.pml_width;
  return P->ew_on && P->prec == 0 && w > 0 && nx > 2 * w && ny > 2 * w && !P->eta_on && !P->fused && !P->xfuse &&
         P->xwall_extra == 0 && !seam_active(P) && P->mix == 0 && P->d.kernel == WAVE_KERNEL_STREAM &&
         !ablation_shape() && !getenv("WAVE25_INNER_TILE");
}

// the wall regions of an embedded-wall launch over the z ranges `zr`: x walls
// over the full y range (corners included), y walls over the inner x range,
// 16 x 8 tiles, z-chunks of ew_cz planes, units chunk-major
static bool attach_walls(wave_plan* P, Launch* L, const std::vector<ZRange>& zr, int set) {
  const int nx = (int)P->d.nx, ny = (int)P->d.ny, w = P->d.pml_width;
  StreamParams::Ew& E = L->p.ew;
  int nzmax = 0;
  for (const ZRange& z : zr) nzmax = std::max(nzmax, z.z1 - z.z0);
  const int cz = std::max(1, std::min(nzmax, P->ew_cz > 0 ? P->ew_cz : std::max(8, L->p.cz / 3)));
  const std::array<int, 4> xy[4] = {{0, w, 0, ny}, {nx - w, nx, 0, ny}, {w, nx - w, 0, w}, {w, nx - w, ny - w, ny}};
  E.nreg = 0;
  int tiles = 0, nzc = -1;
  for (const ZRange& z : zr)
    for (const auto& b : xy) {
      if (b[1] <= b[0] || b[3] <= b[2] || z.z1 <= z.z0) continue;
      if (E.nreg == EW_MAX_REG) return false;
      Region& g = E.reg[E.nreg++];
      g.x0 = b[0]; g.x1 = b[1]; g.y0 = b[2]; g.y1 = b[3]; g.z0 = z.z0; g.z1 = z.z1;
      g.ax0 = b[0] & ~3;
      g.ntx = (b[1] - g.ax0 + EW_CW - 1) / EW_CW;
      g.nty = (b[3] - b[2] + EW_TY - 1) / EW_TY;
      g.nzc = (z.z1 - z.z0 + cz - 1) / cz;
      if (nzc >= 0 && g.nzc != nzc) return false;           // (one chunk count per launch)
      nzc = g.nzc;
      g.blk0 = tiles;
      tiles += g.ntx * g.nty;
    }
  if (E.nreg == 0) return false;
  E.cz = cz;
  E.ntile = tiles;
  E.nunits = tiles * nzc;
  E.min_rem = P->ew_rem >= 0 ? P->ew_rem : cz;
  E.last_blk = std::max(0, L->nblk - P->occ[KI_EW] * P->nsm);
  E.ctr = P->ew_ctr + 2 * set;
  E.pf = P->ew_pf;
  E.dbg = P->ew_dbg;
  return true;
}

static wave_status build_launches(wave_plan* P) {
  const int nx = (int)P->d.nx, ny = (int)P->d.ny, nz = (int)P->d.nz, w = P->d.pml_width;
  std::vector<ZRange> all = {{0, nz}}, edges, inter;
  if (nz <= 2 * R) {
    edges = all;
  } else {
    edges = {{0, R}, {nz - R, nz}};
    inter = {{R, nz - R}};
  }
  const std::vector<ZRange>* sets[3] = {&all, &edges, &inter};
  for (int s = 0; s < 3; ++s) {
    P->launches[s].clear();
    if (sets[s]->empty()) continue;
    if (P->fused) {
      // one launch over the whole plane, path per warp
      add_regions(P, KI_FUSED, {{0, nx, 0, ny}}, *sets[s], &P->launches[s]);
      continue;
    }
    if (P->xfuse && !P->eta_on) {
      // x walls inside the (fused-mode) interior tiles over the full x range;
      // y walls (corners included) over the full x range
      add_regions(P, KI_FUSED, {{0, nx, w, ny - w}}, *sets[s], &P->launches[s]);
      if (w > 0) add_regions(P, KI_WALLY, {{0, nx, 0, w}, {0, nx, ny - w, ny}}, *sets[s], &P->launches[s]);
      continue;
    }
    // embedded walls: one launch, the interior tiles' CTAs
    // compute the four PML walls in their spare warps
    if (ew_wanted(P)) {
      std::vector<Launch> tmp;
      add_regions(P, KI_EW, {{w, nx - w, w, ny - w}}, *sets[s], &tmp);
      if (tmp.size() == 1 && attach_walls(P, &tmp[0], *sets[s], s)) {
        P->launches[s].push_back(tmp[0]);
        continue;
      }
    }
    // interior kernel: inner xy footprint, all z (z caps plane-uniform); with a
    // stored eta the caps are not plane-uniform and go to the wall kernel
    if (P->eta_on && s == 0 && nz > 2 * w) {
      add_regions(P, KI_INNER, {{w, nx - w, w, ny - w}}, {{w, nz - w}}, &P->launches[s]);
      if (w > 0)
        add_regions(P, KI_WALLY_E, {{w, nx - w, w, ny - w}}, {{0, w}, {nz - w, nz}}, &P->launches[s]);
    } else if (P->eta_on && s == 0) {
      add_regions(P, KI_WALLY_E, {{w, nx - w, w, ny - w}}, *sets[s], &P->launches[s]);
    } else {
      const int xw = w > 0 ? w + P->xwall_extra : 0;
      add_regions(P, KI_INNER, {{xw, nx - xw, w, ny - w}}, *sets[s], &P->launches[s]);
    }
    // boundary kernels: left/right (x) walls over the full y range (corners
    // included); front/back (y) walls over the inner x range, so that their
    // tiles line up with the interior kernel's wide tiles
    if (w > 0) {
      const int kx = P->eta_on ? KI_WALLX_E : KI_WALLX, ky = P->eta_on ? KI_WALLY_E : KI_WALLY;
      // x-wall width (>= w: extra inner columns; not with a stored eta, whose
      // interior launch keeps the inner xy footprint)
      const int xw = w + (P->eta_on ? 0 : P->xwall_extra);
      if (seam_active(P))   // both x walls as seams t = 0..ny (x range [R, R + 2w) of the seam views)
        add_regions(P, KI_SEAM, {{R, R + 2 * w, 0, ny + 1}}, *sets[s], &P->launches[s]);
      else
        add_regions(P, kx, {{0, xw, 0, ny}, {nx - xw, nx, 0, ny}}, *sets[s], &P->launches[s]);
      add_regions(P, ky, {{xw, nx - xw, 0, w}, {xw, nx - xw, ny - w, ny}}, *sets[s], &P->launches[s]);
    }
  }
  // interior + x walls as one grid (k_mix): the x-wall launch
  // takes the interior's z-chunks; chunk by chunk, the wall tiles go next to
  // the interior tile rows they border
  P->mix_ok = false;
  if (P->mix && P->prec == 0 && !P->eta_on && !P->fused && !P->xfuse && P->xwall_extra == 0 && w > 0 &&
      P->kt[KI_INNER].fn == mix_inner().fn && P->kt[KI_WALLX].fn == mix_wallx().fn) {
    Launch* Li = nullptr;
    Launch* Lx = nullptr;
    for (Launch& L : P->launches[0]) {
      if (L.ki == KI_INNER) Li = Li ? nullptr : &L;
      if (L.ki == KI_WALLX) Lx = Lx ? nullptr : &L;
    }
    if (Li && Lx && Li->p.nreg == 1 && Lx->p.nreg == 2) {
      const Region& gi = Li->p.reg[0];
      StreamParams& pw = Lx->p;
      const int cz = Li->p.cz, ncw = pw.reg[0].ntx * pw.reg[0].nty;
      bool ok = pw.reg[1].ntx * pw.reg[1].nty == ncw && pw.reg[0].ntx == 1;
      int blk = 0;
      for (int r = 0; r < 2 && ok; ++r) {
        Region& g = pw.reg[r];
        ok = g.z0 == gi.z0 && g.z1 == gi.z1;
        g.nzc = (g.z1 - g.z0 + cz - 1) / cz;
        g.blk0 = blk;
        blk += ncw * g.nzc;
      }
      if (ok && pw.reg[0].nzc == gi.nzc) {
        pw.cz = cz;
        pw.inter2 = 0;
        Lx->nblk = blk;
        // chunk sequence: interior tiles in tile-row order; wall tile t of
        // each side right after the interior row holding its middle y
        const int ni = gi.ntx * gi.nty;
        std::vector<std::vector<int>> after(gi.nty);
        for (int r = 0; r < 2; ++r)
          for (int t = 0; t < ncw; ++t) {
            const int ymid = pw.reg[r].y0 + t * g_k[0][KI_WALLX].ty + g_k[0][KI_WALLX].ty / 2;
            const int row = std::max(0, std::min(gi.nty - 1, (ymid - gi.y0) / P->kt[KI_INNER].ty));
            after[row].push_back(-(1 + r * ncw + t));
          }
        std::vector<int> seq;
        if (P->mix == 2)                  // WAVE25_MIX=2: every wall tile at the start of its chunk
          for (int row = 0; row < gi.nty; ++row) { seq.insert(seq.end(), after[row].begin(), after[row].end()); after[row].clear(); }
        for (int row = 0; row < gi.nty; ++row) {
          for (int tx = 0; tx < gi.ntx; ++tx) seq.push_back(row * gi.ntx + tx);
          for (int q : after[row]) seq.push_back(q);
        }
        if (P->mix_seq_d) { cudaFree(P->mix_seq_d); P->mix_seq_d = nullptr; }
        CK(cudaMalloc(&P->mix_seq_d, seq.size() * sizeof(int)));
        CK(cudaMemcpy(P->mix_seq_d, seq.data(), seq.size() * sizeof(int), cudaMemcpyHostToDevice));
        P->mixp.pi = Li->p;
        P->mixp.pw = pw;
        P->mixp.seq = P->mix_seq_d;
        P->mixp.per_chunk = (int)seq.size();
        P->mixp.ni = ni;
        P->mix_nblk = (int)seq.size() * gi.nzc;
        P->mix_ok = true;
      }
    }
  }
  // two-step temporal blocking: interior launch over the (w+4)-shrunk inner xy
  // box, walls in two single-step phases over frames of width w+8 and w+4
  // two steps through L2: one launch over the inner xy footprint x all z,
  // whole-z columns, 2 blocks per tile (step 1, step 2) in dependency order
  P->pair_ok = false;
  if (P->d.kernel == WAVE_KERNEL_PAIR && P->d.nz == P->d.nz_global && !P->eta_on && nx > 2 * w && ny > 2 * w) {
    std::vector<Launch> tmp;
    add_regions(P, KI_PAIR, {{w, nx - w, w, ny - w}}, all, &tmp);
    if (tmp.size() == 1 && tmp[0].p.nreg == 1 && tmp[0].p.reg[0].nty < 65536 && (nz + 7) / 8 < 4096) {
      Launch L = tmp[0];
      Region& g = L.p.reg[0];
      // z chunks of pair_cz planes (>= 8): short blocks keep step 2 close behind
      // step 1 in time, so u^{n+1}, u^n and vdt2 are still in L2 when it reads them
      const int cz = std::max(8, std::min(P->pair_cz, nz));
      const int nzc = (nz + cz - 1) / cz;
      L.p.cz = cz;
      g.nzc = nzc;
      g.blk0 = 0;
      const int nrow = g.nty;
      std::vector<int> groups;              // role << 28 | chunk << 16 | tile row, dependency order
      for (int k = 0; k < nzc; ++k) {
        groups.push_back((1 << 28) | (k << 16) | 0);
        for (int r = 0; r < nrow; ++r) {
          if (r + 1 < nrow) groups.push_back((1 << 28) | (k << 16) | (r + 1));
          groups.push_back((2 << 28) | (k << 16) | r);
        }
      }
      L.nblk = (int)groups.size() * g.ntx;
      L.p.pf = 0;
      const int64_t ntile = (int64_t)g.ntx * g.nty * nzc;
      if (P->pair_groups_d) { cudaFree(P->pair_groups_d); P->pair_groups_d = nullptr; }
      if (P->prog_d) { cudaFree(P->prog_d); P->prog_d = nullptr; }
      CK(cudaMalloc(&P->pair_groups_d, groups.size() * sizeof(int)));
      CK(cudaMemcpy(P->pair_groups_d, groups.data(), groups.size() * sizeof(int), cudaMemcpyHostToDevice));
      const int64_t ndbg = (P->pair_dbg & 8) ? 12 * (int64_t)L.nblk + 2 : 0;   // u32 words, u64-aligned
      L.p.pair_ticket = ntile;                              // after the per-tile counters
      L.p.pair_dbg_off = (ntile + 2) & ~(int64_t)1;
      CK(cudaMalloc(&P->prog_d, (L.p.pair_dbg_off + ndbg) * sizeof(unsigned)));
      P->prog_n = ntile + 1;                                // counters + ticket, zeroed per launch
      L.p.pair_groups = P->pair_groups_d;
      L.p.prog = P->prog_d;
      P->pair_launch = L;
      P->pair_ok = true;
    }
  }
  P->wall_p1.clear();
  P->wall_p2.clear();
  P->t2_ok = false;
  if (P->d.kernel == WAVE_KERNEL_TB2 && P->d.nz == P->d.nz_global && nx >= 2 * w + 17 && ny >= 2 * w + 17) {
    const T2Info& T = P->t2;
    T2Params& q = P->t2p;
    memset(&q, 0, sizeof q);
    q.pitch = P->L.pitch_x;
    q.plane = P->L.pitch_x * P->d.ny;
    q.nx = nx; q.ny = ny; q.nzl = nz; q.nzg = (int)P->d.nz_global; q.zoff = 0; q.w = w;
    q.dx0 = w + 4; q.dx1 = nx - w - 4; q.dy0 = w + 4; q.dy1 = ny - w - 4;   // u^{n+2} box
    q.cx0 = w + 8; q.cx1 = nx - w - 8; q.cy0 = w + 8; q.cy1 = ny - w - 8;   // u^{n+1} box
    q.ax0 = q.dx0 & ~3;
    q.ay0 = q.dy0;
    q.ntx = (q.dx1 - q.ax0 + T.tx - 1) / T.tx;
    q.nty = (q.dy1 - q.ay0 + T.ty - 1) / T.ty;
    int cz = choose_cz((int64_t)q.ntx * q.nty, nz, P->occ_t2 * P->nsm, 8.0);
    if (const char* e = getenv("WAVE25_T2_CZ")) cz = std::max(1, std::min(nz, atoi(e)));
    q.cz = cz;
    q.nzc = (nz + cz - 1) / cz;
    q.k = P->coef;
    q.tab = static_cast<const float*>(P->tab_d);
    q.sk = -1;
    P->t2_nblk = q.ntx * q.nty * q.nzc;
    const int f1 = w + 8, f2 = w + 4;
    add_regions(P, KI_WALLX, {{0, f1, f1, ny - f1}, {nx - f1, nx, f1, ny - f1}}, all, &P->wall_p1);
    add_regions(P, KI_WALLY, {{0, nx, 0, f1}, {0, nx, ny - f1, ny}}, all, &P->wall_p1);
    add_regions(P, KI_WALLX, {{0, f2, f2, ny - f2}, {nx - f2, nx, f2, ny - f2}}, all, &P->wall_p2);
    add_regions(P, KI_WALLY, {{0, nx, 0, f2}, {0, nx, ny - f2, ny}}, all, &P->wall_p2);
    P->t2_ok = true;
  }
  return WAVE_OK;
}

static void add_regions(wave_plan* P, int ki, const std::vector<std::array<int, 4>>& xy,
                        const std::vector<ZRange>& zr, std::vector<Launch>* out) {
  const int CW = KCW(ki), TY = KTY(ki), CLS = KCL(ki);
  // chunk length from the largest z range and the total column count
  int64_t ncol = 0;
  int nzmax = 0;
  for (auto& b : xy) {
    if (b[1] <= b[0] || b[3] <= b[2]) continue;
    const int ax0 = b[0] & ~3;
    ncol += (int64_t)((b[1] - ax0 + CW - 1) / CW) * ((b[3] - b[2] + TY - 1) / TY);
  }
  for (auto& z : zr) nzmax = std::max(nzmax, z.z1 - z.z0);
  if (ncol == 0 || nzmax == 0) return;
  const int resident = P->occ[ki] * P->nsm;
  // fp32 wall kernels: chunks of at most W25_WALL_CZ_MAX planes, so that the
  // short wall CTAs interleave with the interior's instead of holding most SMs
  // for one long wave (C3: 2.88 -> 2.83 ms/step; C2 keeps its one-wave 29
  // planes; DESIGN.md §5 ablation, profiles/wallcz_r01.txt)
  const int maxcz = (P->prec == 0 && (ki == KI_WALLX || ki == KI_WALLY)) ? W25_WALL_CZ_MAX : (1 << 30);
  int cz = choose_cz(ncol * (int64_t)zr.size(), nzmax, resident, 4.0, maxcz);
  if (ki == KI_INNER)
    if (const char* e = getenv("WAVE25_CZ")) cz = std::max(1, std::min(nzmax, atoi(e)));
  if (is_wall(ki) && P->wall_cz > 0) cz = std::min(nzmax, P->wall_cz);

  Launch Lc;
  Lc.ki = ki;
  StreamParams& p = Lc.p;
  memset(&p, 0, sizeof p);
  p.pitch = P->L.pitch_x;
  p.plane = P->L.pitch_x * P->d.ny;
  p.nx = (int)P->d.nx; p.ny = (int)P->d.ny; p.nzl = (int)P->d.nz;
  p.nzg = (int)P->d.nz_global; p.zoff = (int)P->d.z_offset; p.w = P->d.pml_width;
  p.k = P->coef;
  p.kd = P->coefd;
  p.tab = P->tab_d;
  p.fastdiv = P->fastdiv ? 1 : 0;
  p.eta = P->eta_on ? P->eta_buf : nullptr;
  if (P->eta_on && (ki == KI_WALLX_E || ki == KI_WALLY_E)) {
    // the stored eta, staged through the u_prev/vdt2 ring: box (CW + 8) x (TY + 2)
    const uint64_t pb = P->L.pitch_x * 4;
    encode3d(&p.tm_eta, P->eta_buf, P->d.nx, P->d.ny, P->d.nz, pb, pb * P->d.ny, CW + 8, TY + 2, false);
  }
  p.dt = (double)P->dt;
  p.cz = cz;
  p.pf = (is_wall(ki) && P->wall_pf >= 0) ? P->wall_pf : P->pf;
  p.order = P->order;
  p.upol = P->upol;
  p.st_keep = (is_wall(ki) && P->wall_keep) ? 1 : 0;
  int blk = 0;
  auto flush = [&]() {
    if (p.nreg == 0) return;
    Lc.nblk = blk;
    out->push_back(Lc);
    p.nreg = 0;
    blk = 0;
  };
  for (auto& z : zr) {
    for (auto& b : xy) {
      if (b[1] <= b[0] || b[3] <= b[2] || z.z1 <= z.z0) continue;
      if (p.nreg == MAX_REGIONS) flush();
      Region& g = p.reg[p.nreg++];
      g.x0 = b[0]; g.x1 = b[1]; g.y0 = b[2]; g.y1 = b[3]; g.z0 = z.z0; g.z1 = z.z1;
      g.ax0 = b[0] & ~3;
      g.ntx = (b[1] - g.ax0 + CW - 1) / CW;
      g.nty = (b[3] - b[2] + TY - 1) / TY;
      g.nty = (g.nty + CLS - 1) / CLS * CLS;     // whole clusters (rows beyond y1 are masked)
      g.nzc = (z.z1 - z.z0 + cz - 1) / cz;
      g.blk0 = blk;
      blk += g.ntx * g.nty * g.nzc;
    }
  }
  flush();
  // the two x walls of one z range: interleave their blocks, so that the left
  // wall of row y+1 and the right wall of row y -- one 128-B line with the
  // origin shift -- are streamed by concurrent CTAs (one DRAM fetch)
  if (ki == KI_WALLX && P->xinter && !out->empty() && out->back().ki == KI_WALLX) {
    Launch& L = out->back();
    StreamParams& q = L.p;
    if (q.nreg == 2 && q.reg[0].ntx * q.reg[0].nty * q.reg[0].nzc == q.reg[1].ntx * q.reg[1].nty * q.reg[1].nzc)
      q.inter2 = 1;
  }
}

// ---------------------------------------------------------------------------
// step enqueue
// ---------------------------------------------------------------------------
// Code-shape ablation: WAVE25_ABLATION replaces the interior
// kernel by one of the paper's shapes (paper_shapes.cuh) over the same regions.
static const char* ablation_shape() {
  static const char* e = getenv("WAVE25_ABLATION");
  return (e && *e) ? e : nullptr;
}

template <bool CHK>
static bool launch_shape(const char* sh, const AblParams& a, int ex, int ey, int ez, cudaStream_t s) {
  auto cdiv = [](int a_, int b_) { return (unsigned)((a_ + b_ - 1) / b_); };
  if (!strcmp(sh, "gmem_32x4x1")) k_gmem<32, 4, 1, CHK><<<dim3(cdiv(ex, 32), cdiv(ey, 4), ez), dim3(32, 4, 1), 0, s>>>(a);
  else if (!strcmp(sh, "gmem_8x8x8")) k_gmem<8, 8, 8, CHK><<<dim3(cdiv(ex, 8), cdiv(ey, 8), cdiv(ez, 8)), dim3(8, 8, 8), 0, s>>>(a);
  else if (!strcmp(sh, "smem_u")) k_smem_u<CHK><<<dim3(cdiv(ex, 8), cdiv(ey, 8), cdiv(ez, 8)), dim3(8, 8, 8), 0, s>>>(a);
  else if (!strcmp(sh, "st_smem_32x16")) k_st<ST_SMEM, 32, 16, CHK><<<dim3(cdiv(ex, 32), cdiv(ey, 16)), dim3(32, 16), 0, s>>>(a);
  else if (!strcmp(sh, "st_reg_shft_32x16")) k_st<ST_SHFT, 32, 16, CHK><<<dim3(cdiv(ex, 32), cdiv(ey, 16)), dim3(32, 16), 0, s>>>(a);
  else if (!strcmp(sh, "st_reg_fixed_32x16")) k_st<ST_FIXED, 32, 16, CHK><<<dim3(cdiv(ex, 32), cdiv(ey, 16)), dim3(32, 16), 0, s>>>(a);
  else if (!strcmp(sh, "st_reg_fixed_32x32")) k_st<ST_FIXED, 32, 32, CHK><<<dim3(cdiv(ex, 32), cdiv(ey, 32)), dim3(32, 32), 0, s>>>(a);
  else if (!strcmp(sh, "semi_32x16")) k_semi<32, 16, CHK><<<dim3(cdiv(ex, 32), cdiv(ey, 16)), dim3(32, 16), 0, s>>>(a);
  else return false;
  return true;
}

static wave_status launch_ablation(wave_plan* P, const Launch& Lc, int ui, int upi, float* out, cudaStream_t s) {
  const char* sh = ablation_shape();
  for (int r = 0; r < Lc.p.nreg; ++r) {
    const Region& g = Lc.p.reg[r];
    AblParams a;
    a.u = P->buf[ui]; a.up = P->buf[upi]; a.out = out; a.v = P->vdt2;
    a.pitch = P->L.pitch_x; a.plane = P->L.pitch_x * P->d.ny;
    a.nx = (int)P->d.nx; a.ny = (int)P->d.ny; a.nzl = (int)P->d.nz; a.nzg = (int)P->d.nz_global;
    a.zoff = (int)P->d.z_offset; a.w = P->d.pml_width;
    a.x0 = g.x0; a.x1 = g.x1; a.y0 = g.y0; a.y1 = g.y1; a.z0 = g.z0; a.z1 = g.z1;
    a.k = P->coef; a.tab = static_cast<const float*>(P->tab_d);
    const int ex = g.x1 - g.x0, ey = g.y1 - g.y0, ez = g.z1 - g.z0;
    if (a.w < R) {
      if (!launch_shape<true>(sh, a, ex, ey, ez, s)) return fail(WAVE_ERR_CONFIG, "unknown WAVE25_ABLATION shape '%s'", sh);
    } else if (!launch_shape<false>(sh, a, ex, ey, ez, s)) {
      return fail(WAVE_ERR_CONFIG, "unknown WAVE25_ABLATION shape '%s'", sh);
    }
    CK(cudaGetLastError());
  }
  return WAVE_OK;
}

// u^n in buffer ui, u^{n-1} in buffer upi, u^{n+1} written to `out` (= buf[upi]
// for an in-place step)
static wave_status launch_stream(wave_plan* P, const Launch& Lc, int ui, int upi, float* out, cudaStream_t s) {
  if (Lc.ki == KI_INNER && ablation_shape() && !P->remote && P->prec == 0)
    return launch_ablation(P, Lc, ui, upi, out, s);
  const Maps& M = P->maps[Lc.ki];
  StreamParams p = Lc.p;
  p.out = out;
  p.rlo = p.rhi = nullptr;
  if (P->remote) {
    const int64_t plane = P->L.pitch_x * P->d.ny;
    if (P->peers.lo_buf[upi]) p.rlo = eo(P, P->peers.lo_buf[upi], (P->peers.lo_nz + R) * plane);
    if (P->peers.hi_buf[upi]) p.rhi = P->peers.hi_buf[upi];
  }
  if (Lc.ki == KI_EW) {
    p.ew.tu = P->maps[KI_EWALL].u[ui];
    p.ew.tup = P->maps[KI_EWALL].up[upi];
    p.ew.tv = P->maps[KI_EWALL].v;
  }
  const dim3 grid(Lc.nblk), block(kernel_threads(P, Lc.ki));
  const size_t smem = kernel_smem(P, Lc.ki);
  if (P->gmaps && P->maps_g) {
    p.gu = &P->maps_g[Lc.ki].u[ui];
    p.gup = &P->maps_g[Lc.ki].up[upi];
    p.gv = &P->maps_g[Lc.ki].v;
  }
  void* args[] = {(void*)&M.u[ui], (void*)&M.up[upi], (void*)&M.v, (void*)&p};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  // wall CTAs (compute-heavy) get priority so they interleave with the
  // bandwidth-bound interior CTAs instead of trailing them
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = (Lc.ki != KI_INNER && Lc.ki != KI_FUSED && P->wall_prio) ? P->prio_hi : P->prio_lo;
  int na = 1;
  if (KCL(Lc.ki) > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = KCL(Lc.ki);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (P->l2_persist_mb > 0) {
    // L2 set-aside for u^n: its lines (re-read as neighbours' halos) persist,
    // u_prev / vdt2 / u_next stream through the rest of L2
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow.base_ptr = P->buf[ui];
    attr[na].val.accessPolicyWindow.num_bytes = std::min<size_t>(P->L.elems_u * 4, P->max_window);
    attr[na].val.accessPolicyWindow.hitRatio = P->l2_hit_ratio;
    attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CK(cudaLaunchKernelExC(&cfg, kernel_ptr(P, Lc.ki), args));
  return WAVE_OK;
}

// interior + x walls in one grid
static bool mix_active(const wave_plan* P) {
  return P->mix_ok && !P->remote && !(P->gmaps && P->maps_g) && P->l2_persist_mb == 0 && !ablation_shape();
}

static wave_status launch_mix(wave_plan* P, int ui, int upi, float* out, cudaStream_t s) {
  const Maps& Mi = P->maps[KI_INNER];
  const Maps& Mw = P->maps[KI_WALLX];
  MixParams m = P->mixp;
  m.pi.out = m.pw.out = out;
  m.pi.rlo = m.pi.rhi = m.pw.rlo = m.pw.rhi = nullptr;
  void* args[] = {(void*)&Mi.u[ui], (void*)&Mi.up[upi], (void*)&Mi.v,
                  (void*)&Mw.u[ui], (void*)&Mw.up[upi], (void*)&Mw.v, (void*)&m};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->mix_nblk);
  cfg.blockDim = dim3(kernel_threads(P, KI_INNER));
  cfg.dynamicSmemBytes = std::max(kernel_smem(P, KI_INNER), kernel_smem(P, KI_WALLX));
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = P->prio_lo;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelExC(&cfg, mix_fn(), args));
  return WAVE_OK;
}

static wave_status launch_naive(wave_plan* P, int cur, int prv, int z0, int z1, cudaStream_t s) {
  if (z1 <= z0) return WAVE_OK;
  NaiveParams np;
  np.pitch = P->L.pitch_x;
  np.plane = P->L.pitch_x * P->d.ny;
  np.nx = (int)P->d.nx; np.ny = (int)P->d.ny; np.nzl = (int)P->d.nz;
  np.nzg = (int)P->d.nz_global; np.zoff = (int)P->d.z_offset; np.w = P->d.pml_width;
  np.z0 = z0;
  np.k = P->coef;
  np.kd = P->coefd;
  np.tab = P->tab_d;
  np.eta = P->eta_on ? P->eta_buf : nullptr;
  np.dt = (double)P->dt;
  const dim3 grid((unsigned)((P->d.nx + 31) / 32), (unsigned)((P->d.ny + 3) / 4), (unsigned)(z1 - z0));
  if (P->prec)
    k_naive<double><<<grid, dim3(32, 4), 0, s>>>(reinterpret_cast<const double*>(P->buf[cur]),
                                                 reinterpret_cast<double*>(P->buf[prv]),
                                                 reinterpret_cast<const double*>(P->vdt2), np);
  else
    k_naive<float><<<grid, dim3(32, 4), 0, s>>>(P->buf[cur], P->buf[prv], P->vdt2, np);
  CK(cudaGetLastError());
  return WAVE_OK;
}

// source into u^{n+1} = buf[prv] after an in-place step; advances the device step counter
static wave_status launch_source(wave_plan* P, int prv, cudaStream_t s) {
  if (!P->src_set || !P->src_local || P->ninc == 0) return WAVE_OK;
  const int64_t k = P->sk - P->d.z_offset;
  const int64_t plane = P->L.pitch_x * P->d.ny;
  const int64_t off = (k + R) * plane + P->sj * P->L.pitch_x + P->si;
  // the source cell in the neighbours' ghost planes (fused exchange); both
  // mirrors are independent (a plane of a thin slab can be an edge of both faces)
  float* mlo = nullptr;
  float* mhi = nullptr;
  if (P->remote) {
    const int64_t cell = P->sj * P->L.pitch_x + P->si;
    if (k < R && P->peers.lo_buf[prv]) mlo = eo(P, P->peers.lo_buf[prv], (P->peers.lo_nz + R + k) * plane + cell);
    if (k >= P->d.nz - R && P->peers.hi_buf[prv]) mhi = eo(P, P->peers.hi_buf[prv], (k - (P->d.nz - R)) * plane + cell);
  }
  if (P->prec)
    k_source<double><<<1, 1, 0, s>>>(reinterpret_cast<double*>(P->buf[prv]), off,
                                     static_cast<const double*>(P->inc_d), P->ninc, P->dstep,
                                     reinterpret_cast<double*>(mlo), reinterpret_cast<double*>(mhi));
  else
    k_source<float><<<1, 1, 0, s>>>(P->buf[prv], off, static_cast<const float*>(P->inc_d), P->ninc, P->dstep,
                                    mlo, mhi);
  CK(cudaGetLastError());
  return WAVE_OK;
}

// which: 0 all planes, 1 edges, 2 interior
static wave_status enqueue_compute(wave_plan* P, int which, int cur, int prv, cudaStream_t s) {
  if (P->d.kernel == WAVE_KERNEL_NAIVE) {
    const int nz = (int)P->d.nz;
    if (which == 0 || (which == 1 && nz <= 2 * R)) return launch_naive(P, cur, prv, 0, nz, s);
    if (which == 1) {
      CKST(launch_naive(P, cur, prv, 0, R, s));
      return launch_naive(P, cur, prv, nz - R, nz, s);
    }
    return nz <= 2 * R ? WAVE_OK : launch_naive(P, cur, prv, R, nz - R, s);
  }
  const std::vector<Launch>& Ls = P->launches[which];
  if (Ls.empty()) return WAVE_OK;
  const bool mix = which == 0 && mix_active(P);
  auto mixed_out = [&](int ki) { return mix && (ki == KI_INNER || ki == KI_WALLX); };
  // fork BEFORE any launch: the wall kernels (side stream, high priority) and
  // the interior kernel (stream s) run concurrently; join before the source
  bool walls = false;
  for (const Launch& L : Ls) walls |= is_wall(L.ki);
  if (walls && P->serial) {                 // WAVE25_SERIAL=1: everything on `s`, walls first
    for (const Launch& L : Ls)
      if (is_wall(L.ki) && !mixed_out(L.ki)) CKST(launch_stream(P, L, cur, prv, P->buf[prv], s));
    walls = false;
  }
  auto launch_walls = [&]() -> wave_status {
    for (const Launch& L : Ls)
      if (is_wall(L.ki) && !mixed_out(L.ki)) {
        const bool y = L.ki == KI_WALLY || L.ki == KI_WALLY_E;
        CKST(launch_stream(P, L, cur, prv, P->buf[prv], (y && P->side2_on) ? P->side2 : P->side));
      }
    return WAVE_OK;
  };
  if (walls) {
    CK(cudaEventRecord(P->ev_fork, s));
    CK(cudaStreamWaitEvent(P->side, P->ev_fork, 0));
    if (P->side2_on) CK(cudaStreamWaitEvent(P->side2, P->ev_fork, 0));
    if (!P->walls_last) CKST(launch_walls());
  }
  if (mix) CKST(launch_mix(P, cur, prv, P->buf[prv], s));
  for (const Launch& L : Ls)
    if (!is_wall(L.ki) && !mixed_out(L.ki)) CKST(launch_stream(P, L, cur, prv, P->buf[prv], s));
  if (walls && P->walls_last) CKST(launch_walls());
  if (P->serial) return WAVE_OK;
  if (walls) {
    CK(cudaEventRecord(P->ev_join, P->side));
    CK(cudaStreamWaitEvent(s, P->ev_join, 0));
    if (P->side2_on) {
      CK(cudaEventRecord(P->ev_join2, P->side2));
      CK(cudaStreamWaitEvent(s, P->ev_join2, 0));
    }
  }
  return WAVE_OK;
}

static bool source_in(const wave_plan* P, int which) {
  if (!P->src_set || !P->src_local) return false;
  const int64_t k = P->sk - P->d.z_offset, nz = P->d.nz;
  if (which == 0) return true;
  const bool edge = nz <= 2 * R || k < R || k >= nz - R;
  return which == 1 ? edge : !edge;
}

// one in-place step: u^{n+1} into buf[prv]
static wave_status enqueue_step(wave_plan* P, int cur, int prv, cudaStream_t s) {
  CKST(enqueue_compute(P, 0, cur, prv, s));
  return launch_source(P, prv, s);
}

static wave_status capture(wave_plan* P, cudaGraphExec_t* out, wave_status (*body)(wave_plan*, int, int),
                           int cur, int prv) {
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(P->cap, cudaStreamCaptureModeThreadLocal));
  wave_status st = body(P, cur, prv);
  cudaError_t e = cudaStreamEndCapture(P->cap, &g);
  if (st != WAVE_OK) { if (g) cudaGraphDestroy(g); return st; }
  if (e != cudaSuccess) return fail(WAVE_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(WAVE_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  return WAVE_OK;
}

static wave_status two_single_steps(wave_plan* P, int cur, int prv) {
  if (P->walls_alt) {
    // walls after the interior in the first step, before it in the second: the
    // two wall phases are adjacent in time, so the second reads the wall data
    // the first just wrote / read from L2 (A/B)
    const bool keep = P->walls_last;
    P->walls_last = true;
    wave_status st = enqueue_step(P, cur, prv, P->cap);
    P->walls_last = false;
    if (st == WAVE_OK) st = enqueue_step(P, prv, cur, P->cap);
    P->walls_last = keep;
    return st;
  }
  CKST(enqueue_step(P, cur, prv, P->cap));
  return enqueue_step(P, prv, cur, P->cap);
}

// a 2-step graph of single steps returns to the same (cur, prv)
static wave_status ensure_graph(wave_plan* P, int cur, int prv) {
  cudaGraphExec_t* g = &P->gexec[cur * 4 + prv];
  return *g ? WAVE_OK : capture(P, g, two_single_steps, cur, prv);
}

// ---------------------------------------------------------------------------
// two-step temporal blocking (WAVE_KERNEL_TB2, tb2.cuh)
// ---------------------------------------------------------------------------
static bool tb2_active(const wave_plan* P) {
  return P->d.kernel == WAVE_KERNEL_TB2 && P->aux && P->t2_ok && !P->eta_on;
}

// the two buffers not holding (u^n, u^{n-1}): C gets u^{n+1}, D gets u^{n+2}
static void pair_targets(int cur, int prv, int* c, int* d) {
  int o[2], n = 0;
  for (int b = 0; b < 4; ++b)
    if (b != cur && b != prv) o[n++] = b;
  *c = o[0];
  *d = o[1];
}

static int64_t source_offset(const wave_plan* P) {
  const int64_t k = P->sk - P->d.z_offset;
  return (k + R) * P->L.pitch_x * P->d.ny + P->sj * P->L.pitch_x + P->si;
}

static bool source_active(const wave_plan* P) { return P->src_set && P->src_local && P->ninc > 0; }

// source (x, y) inside the frame of width w + e that the pair's wall kernels compute
static bool source_in_frame(const wave_plan* P, int e) {
  const int64_t w = P->d.pml_width + e;
  return !(P->si >= w && P->si < P->d.nx - w && P->sj >= w && P->sj < P->d.ny - w);
}

static wave_status launch_t2(wave_plan* P, int cur, int prv, int c, int d, cudaStream_t s) {
  T2Params p = P->t2p;
  p.outC = P->buf[c];
  p.outD = P->buf[d];
  p.si = (int)P->si;
  p.sj = (int)P->sj;
  p.sk = source_active(P) ? (int)(P->sk - P->d.z_offset) : -1;
  p.dstep = P->dstep;
  p.inc = static_cast<const float*>(P->inc_d);
  p.ninc = P->ninc;
  void* args[] = {(void*)&P->t2maps.u[cur], (void*)&P->t2maps.up[prv], (void*)&P->t2maps.v1,
                  (void*)&P->t2maps.v2, (void*)&p};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->t2_nblk);
  cfg.blockDim = dim3(P->t2.nt);
  cfg.dynamicSmemBytes = P->t2.smem(P->d.pml_width);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = P->prio_lo;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelExC(&cfg, P->t2.fn, args));
  return WAVE_OK;
}

// One pair: (u^n = buf[cur], u^{n-1} = buf[prv]) -> (u^{n+1} = buf[c], u^{n+2} = buf[d]).
// Interior: one k_tb2 launch.  Walls (side stream, overlapping it): u^{n+1} on
// the (w+8)-wide frame, then u^{n+2} on the (w+4)-wide frame from it -- the
// interior launch needs neither (it recomputes its own halo).
static wave_status enqueue_pair(wave_plan* P, int cur, int prv, cudaStream_t s) {
  int c, d;
  pair_targets(cur, prv, &c, &d);
  const bool src = source_active(P);
  const bool sp1 = src && source_in_frame(P, 8), sp2 = src && source_in_frame(P, 4);
  const bool walls = !P->wall_p1.empty() || !P->wall_p2.empty() || sp1 || sp2;
  if (walls) {
    CK(cudaEventRecord(P->ev_fork, s));
    CK(cudaStreamWaitEvent(P->side, P->ev_fork, 0));
    for (const Launch& L : P->wall_p1) CKST(launch_stream(P, L, cur, prv, P->buf[c], P->side));
    if (sp1) {
      k_source_at<float><<<1, 1, 0, P->side>>>(P->buf[c], source_offset(P), static_cast<const float*>(P->inc_d), P->ninc,
                                        P->dstep, 0);
      CK(cudaGetLastError());
    }
    for (const Launch& L : P->wall_p2) CKST(launch_stream(P, L, c, cur, P->buf[d], P->side));
    if (sp2) {
      k_source_at<float><<<1, 1, 0, P->side>>>(P->buf[d], source_offset(P), static_cast<const float*>(P->inc_d), P->ninc,
                                        P->dstep, 1);
      CK(cudaGetLastError());
    }
  }
  CKST(launch_t2(P, cur, prv, c, d, s));
  if (walls) {
    CK(cudaEventRecord(P->ev_join, P->side));
    CK(cudaStreamWaitEvent(s, P->ev_join, 0));
  }
  if (src) {
    k_advance<<<1, 1, 0, s>>>(P->dstep, 2);
    CK(cudaGetLastError());
  }
  return WAVE_OK;
}

static wave_status one_pair(wave_plan* P, int cur, int prv) { return enqueue_pair(P, cur, prv, P->cap); }

static wave_status ensure_pair_graph(wave_plan* P, int cur, int prv) {
  cudaGraphExec_t* g = &P->gexec2[cur * 4 + prv];
  return *g ? WAVE_OK : capture(P, g, one_pair, cur, prv);
}

// kernel launches of one pair
static int pair_launches(const wave_plan* P) {
  const bool src = source_active(P);
  return 1 + (int)P->wall_p1.size() + (int)P->wall_p2.size() + (src && source_in_frame(P, 8)) +
         (src && source_in_frame(P, 4)) + src;
}

// ---------------------------------------------------------------------------
// two steps through L2 (WAVE_KERNEL_PAIR)
// ---------------------------------------------------------------------------
static bool pair_active(const wave_plan* P) {
  return P->d.kernel == WAVE_KERNEL_PAIR && P->pair_ok && !P->eta_on && P->maps_g;
}

// source inside the PML walls: buf[b] += inc[n + delta] after the wall kernels
// of step n + delta + 1 (the pair kernel injects an interior source itself)
static wave_status pair_wall_source(wave_plan* P, int b, int delta, cudaStream_t s) {
  if (!source_active(P) || !source_in_frame(P, 0)) return WAVE_OK;
  if (P->d.precision == WAVE_PREC_FP64)
    k_source_at<double><<<1, 1, 0, s>>>(reinterpret_cast<double*>(P->buf[b]), source_offset(P),
                                        static_cast<const double*>(P->inc_d), P->ninc, P->dstep, delta);
  else
    k_source_at<float><<<1, 1, 0, s>>>(P->buf[b], source_offset(P), static_cast<const float*>(P->inc_d), P->ninc,
                                       P->dstep, delta);
  CK(cudaGetLastError());
  return WAVE_OK;
}

static wave_status launch_pair_kernel(wave_plan* P, int cur, int prv, cudaStream_t s) {
  const Launch& Lc = P->pair_launch;
  StreamParams p = Lc.p;
  p.gu = &P->maps_g[KI_PAIR].u[cur];        // step 1: u^n = A, u^{n-1} = B -> B
  p.gup = &P->maps_g[KI_PAIR].up[prv];
  p.gv = &P->maps_g[KI_PAIR].v;
  p.out = P->buf[prv];
  p.gu2 = &P->maps_g[KI_PAIR].u[prv];       // step 2: u^{n+1} = B, u^n = A -> A
  p.gup2 = &P->maps_g[KI_PAIR].up[cur];
  p.out2 = P->buf[cur];
  p.rlo = p.rhi = nullptr;
  // a source in the PML walls is added after the wall launches (pair_wall_source)
  const bool src = source_active(P) && !source_in_frame(P, 0);
  p.src_i = (int)P->si;
  p.src_j = (int)P->sj;
  p.src_k = src ? (int)(P->sk - P->d.z_offset) : -1;
  p.inc = P->inc_d;
  p.ninc = P->ninc;
  p.dstep = P->dstep;
  p.pair_dbg = P->pair_dbg;
  p.pair_pk = P->pair_pk;
  const Maps& M = P->maps[KI_PAIR];
  void* args[] = {(void*)&M.u[cur], (void*)&M.up[prv], (void*)&M.v, (void*)&p};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Lc.nblk);
  cfg.blockDim = dim3(kernel_threads(P, KI_PAIR));
  cfg.dynamicSmemBytes = kernel_smem(P, KI_PAIR);
  cfg.stream = s;
  CK(cudaLaunchKernelExC(&cfg, kernel_ptr(P, KI_PAIR), args));
  return WAVE_OK;
}

// One pair: walls step 1 (u^{n+1} on the walls, into B), the interior pair
// kernel (u^{n+1} into B, then u^{n+2} into A, read back through L2), walls
// step 2 (u^{n+2} on the walls, into A).  In place: (cur, prv) unchanged.
static wave_status enqueue_pair_l2(wave_plan* P, int cur, int prv, cudaStream_t s) {
  CK(cudaMemsetAsync(P->prog_d, 0, P->prog_n * sizeof(unsigned), s));
  for (const Launch& L : P->launches[0])
    if (is_wall(L.ki)) CKST(launch_stream(P, L, cur, prv, P->buf[prv], s));
  CKST(pair_wall_source(P, prv, 0, s));
  CKST(launch_pair_kernel(P, cur, prv, s));
  for (const Launch& L : P->launches[0])
    if (is_wall(L.ki)) CKST(launch_stream(P, L, prv, cur, P->buf[cur], s));
  CKST(pair_wall_source(P, cur, 1, s));
  if (source_active(P)) {
    k_advance<<<1, 1, 0, s>>>(P->dstep, 2);
    CK(cudaGetLastError());
  }
  return WAVE_OK;
}

static wave_status one_pair_l2(wave_plan* P, int cur, int prv) { return enqueue_pair_l2(P, cur, prv, P->cap); }

static int pair_l2_launches(const wave_plan* P) {
  int n = 1 + (source_active(P) ? (source_in_frame(P, 0) ? 3 : 1) : 0);
  for (const Launch& L : P->launches[0]) n += is_wall(L.ki) ? 2 : 0;
  return n;
}

static void drop_graphs(wave_plan* P) {
  for (int i = 0; i < 16; ++i) {
    if (P->gexec[i]) { cudaGraphExecDestroy(P->gexec[i]); P->gexec[i] = nullptr; }
    if (P->gexec2[i]) { cudaGraphExecDestroy(P->gexec2[i]); P->gexec2[i] = nullptr; }
    if (P->gexecP[i]) { cudaGraphExecDestroy(P->gexecP[i]); P->gexecP[i] = nullptr; }
  }
  for (int i = 0; i < 2; ++i)
    if (P->gexec_peer[i]) { cudaGraphExecDestroy(P->gexec_peer[i]); P->gexec_peer[i] = nullptr; }
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* wave_version(void) { return "wave25 0.2.0 sm_100a"; }

const char* wave_last_error(void) { return g_err.c_str(); }

wave_status wave_layout(const wave_desc* desc, wave_layout_info* out) {
  CKST(validate(desc));
  if (!out) return fail(WAVE_ERR_CONFIG, "out is NULL");
  make_layout(*desc, out);
  return WAVE_OK;
}

wave_status wave_decompose(const wave_desc* desc, wave_region* out) {
  CKST(validate(desc));
  if (!out) return fail(WAVE_ERR_CONFIG, "out is NULL");
  const int64_t nx = desc->nx, ny = desc->ny, nz = desc->nz_global, w = desc->pml_width;
  auto set = [&](int i, int kind, int64_t x, int64_t y, int64_t z, int64_t ex, int64_t ey, int64_t ez) {
    out[i].kind = kind; out[i].reserved0 = 0;
    out[i].lo[0] = x; out[i].lo[1] = y; out[i].lo[2] = z;
    out[i].ext[0] = ex; out[i].ext[1] = ey; out[i].ext[2] = ez;
  };
  // Inner [w, n-w)^3; Top/Bottom full x,y, z-thickness w; Front/Back full
  // x, y-thickness w, z in [w, nz-w); Left/Right x-thickness w, y in [w, ny-w), z in [w, nz-w)
  set(0, WAVE_REGION_INNER, w, w, w, nx - 2 * w, ny - 2 * w, nz - 2 * w);
  set(1, WAVE_REGION_TOP, 0, 0, 0, nx, ny, w);
  set(2, WAVE_REGION_BOTTOM, 0, 0, nz - w, nx, ny, w);
  set(3, WAVE_REGION_FRONT, 0, 0, w, nx, w, nz - 2 * w);
  set(4, WAVE_REGION_BACK, 0, ny - w, w, nx, w, nz - 2 * w);
  set(5, WAVE_REGION_LEFT, 0, w, w, w, ny - 2 * w, nz - 2 * w);
  set(6, WAVE_REGION_RIGHT, nx - w, w, w, w, ny - 2 * w, nz - 2 * w);
  return WAVE_OK;
}

wave_status wave_constants(const wave_desc* desc, float* c13, float* eta, float* A, float* B,
                           float* inv2h) {
  CKST(validate(desc));
  if (!(desc->dt > 0.f)) return fail(WAVE_ERR_CONFIG, "wave_constants needs dt > 0");
  Coef k;
  std::vector<float> tab;
  make_constants(*desc, desc->dt, &k, &tab);
  const int w = desc->pml_width, T = w + 2;
  if (c13) {
    c13[0] = k.c0;
    for (int m = 0; m < 4; ++m) { c13[1 + m] = k.cx[m]; c13[5 + m] = k.cy[m]; c13[9 + m] = k.cz[m]; }
  }
  for (int d = 0; d <= w; ++d) {
    if (eta) eta[d] = tab[d];
    if (A) A[d] = tab[T + d];
    if (B) B[d] = tab[2 * T + d];
  }
  if (inv2h) for (int a = 0; a < 3; ++a) inv2h[a] = k.i2h[a];
  return WAVE_OK;
}

wave_status wave_division_table(const wave_desc* desc, float* B, float* rB) {
  if (!desc) return fail(WAVE_ERR_CONFIG, "desc is NULL");
  CKST(validate(desc));
  if (!(desc->dt > 0.f)) return fail(WAVE_ERR_CONFIG, "wave_division_table needs desc->dt > 0");
  Coef k;
  std::vector<float> tab;
  make_constants(*desc, desc->dt, &k, &tab);
  const int w = desc->pml_width, T = w + 2;
  for (int d = 0; d <= w; ++d) {
    if (B) B[d] = tab[2 * T + d];
    if (rB) rB[d] = tab[3 * T + d];
  }
  return WAVE_OK;
}

int32_t wave_fastdiv(const wave_plan* P) { return P ? (P->fastdiv ? 1 : 0) : -1; }

wave_status wave_plan_create(const wave_desc* desc, wave_plan** out) {
  CKST(validate(desc));
  if (!out) return fail(WAVE_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  wave_plan* P = new (std::nothrow) wave_plan();
  if (!P) return fail(WAVE_ERR_ALLOC, "host allocation failed");
  P->d = *desc;
  make_layout(P->d, &P->L);
  P->prec = desc->precision == WAVE_PREC_FP64 ? 1 : 0;
  P->esz = P->prec ? 8 : 4;
  P->dt = desc->dt;
  auto bail = [&](wave_status st) { wave_plan_destroy(P); return st; };
  cudaError_t e = cudaGetDevice(&P->dev);
  if (e != cudaSuccess) return bail(fail(WAVE_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e)));
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, P->dev);
  if (major != 10) return bail(fail(WAVE_ERR_CUDA, "this library is built for sm_100a (B200); device is sm_%d*", major));
  cudaDeviceGetAttribute(&P->nsm, cudaDevAttrMultiProcessorCount, P->dev);
  if (get_encoder() != WAVE_OK) return bail(WAVE_ERR_CUDA);
  init_kernels();
  for (int ki = 0; ki < KI_N; ++ki) P->kt[ki] = g_k[P->prec][ki];
  P->kt[KI_INNER] = pick_inner(P->d, P->prec);
  {
    // load every kernel now (lazy module loading can need an idle device,
    // which never comes while a peer-wait kernel spins)
    cudaFuncAttributes fa;
    for (int ki = 0; ki < KI_N; ++ki) cudaFuncGetAttributes(&fa, P->kt[ki].fn);
    const void* aux[] = {(const void*)k_naive<float>, (const void*)k_source<float>, (const void*)k_vdt2<float>,
                         (const void*)k_inc<float>, (const void*)k_stats<float>, (const void*)k_naive<double>,
                         (const void*)k_source<double>, (const void*)k_vdt2<double>, (const void*)k_inc<double>,
                         (const void*)k_stats<double>, (const void*)k_peer_wait, (const void*)k_peer_signal,
                         (const void*)k_copy_planes};
    for (const void* f : aux) cudaFuncGetAttributes(&fa, f);
  }
  if (const char* e = getenv("WAVE25_PF")) P->pf = atoi(e);
  if (const char* e = getenv("WAVE25_PAIR_DBG")) P->pair_dbg = atoi(e);
  if (const char* e = getenv("WAVE25_PAIR_PK")) P->pair_pk = std::max(1, atoi(e));
  if (const char* e = getenv("WAVE25_PAIR_CZ")) P->pair_cz = std::max(8, atoi(e));
  if (const char* e = getenv("WAVE25_WALL_PRIO")) P->wall_prio = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_SERIAL")) P->serial = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_XFUSE")) P->xfuse = atoi(e) != 0;
  // fp32: x walls and y walls on two side streams, concurrently (disjoint
  // output regions; C3 2.841 -> 2.830, C2 0.4224 -> 0.4155 ms/step,
  // profiles/wallsched_r01.txt); WAVE25_SIDE2=0 serialises them on one
  P->side2_on = P->prec == 0;
  if (const char* e = getenv("WAVE25_SIDE2")) P->side2_on = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_WALL_CZ")) P->wall_cz = atoi(e);
  if (const char* e = getenv("WAVE25_XINTER")) P->xinter = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_FASTDIV")) P->fastdiv_on = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_SEAM")) P->seam_on = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_PEER_TIMEOUT_S")) P->peer_timeout_s = std::max(1e-3, atof(e));
  if (const char* e = getenv("WAVE25_XWALL_EXTRA")) P->xwall_extra = std::max(0, atoi(e));
  if (const char* e = getenv("WAVE25_WALLS_LAST")) P->walls_last = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_WALLS_ALT")) P->walls_alt = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_WALL_STKEEP")) P->wall_keep = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_MIX")) P->mix = atoi(e);
  if (const char* e = getenv("WAVE25_WALL_PF")) P->wall_pf = atoi(e);
  if (const char* e = getenv("WAVE25_GMAPS")) P->gmaps = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_ORDER")) P->order = atoi(e);
  if (const char* e = getenv("WAVE25_FUSED")) P->fused = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_UPOL")) P->upol = atoi(e);
  if (const char* e = getenv("WAVE25_EW")) P->ew_on = atoi(e) != 0;
  if (const char* e = getenv("WAVE25_EW_CZ")) P->ew_cz = std::max(1, atoi(e));
  if (const char* e = getenv("WAVE25_EW_REM")) P->ew_rem = atoi(e);
  if (const char* e = getenv("WAVE25_EW_PF")) P->ew_pf = std::max(0, atoi(e));
  if (getenv("WAVE25_EW_DBG") && atoi(getenv("WAVE25_EW_DBG")) != 0) {
    cudaMalloc(&P->ew_dbg, 6 * sizeof(unsigned long long));
    cudaMemset(P->ew_dbg, 0, 6 * sizeof(unsigned long long));
  }
  cudaDeviceGetStreamPriorityRange(&P->prio_lo, &P->prio_hi);
  if (const char* e = getenv("WAVE25_L2MB")) P->l2_persist_mb = atoi(e);
  if (const char* e = getenv("WAVE25_L2HR")) P->l2_hit_ratio = (float)atof(e);
  {
    int mw = 0;
    cudaDeviceGetAttribute(&mw, cudaDevAttrMaxAccessPolicyWindowSize, P->dev);
    P->max_window = (size_t)mw;
  }
  if (P->l2_persist_mb > 0) {
    int mx = 0;
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, P->dev);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>((size_t)P->l2_persist_mb << 20, (size_t)mx));
  }
  const int T = P->d.pml_width + 2;
  if ((e = cudaMalloc(&P->tab_d, 4 * T * P->esz)) != cudaSuccess ||
      (e = cudaMalloc(&P->dstep, sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMalloc(&P->stats_d, sizeof(Stats))) != cudaSuccess ||
      (e = cudaMalloc(&P->ew_ctr, 6 * sizeof(unsigned))) != cudaSuccess ||
      (e = cudaMemset(P->ew_ctr, 0, 6 * sizeof(unsigned))) != cudaSuccess)
    return bail(fail(WAVE_ERR_ALLOC, "cudaMalloc: %s", cudaGetErrorString(e)));
  if ((e = cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&P->cap, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&P->side2, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&P->ev_join2, cudaEventDisableTiming)) != cudaSuccess)
    return bail(fail(WAVE_ERR_CUDA, "stream/event: %s", cudaGetErrorString(e)));
  for (int ki = 0; ki < KI_N; ++ki) {
    const size_t sm = kernel_smem(P, ki);
    if ((e = cudaFuncSetAttribute(kernel_ptr(P, ki), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) != cudaSuccess)
      return bail(fail(WAVE_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(e)));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel_ptr(P, ki), kernel_threads(P, ki), sm);
    P->occ[ki] = std::max(1, occ);
  }
  {
    const size_t sm = std::max(kernel_smem(P, KI_INNER), kernel_smem(P, KI_WALLX));
    if (P->prec == 0 &&
        (e = cudaFuncSetAttribute(mix_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) != cudaSuccess)
      return bail(fail(WAVE_ERR_CUDA, "smem attribute (mix): %s", cudaGetErrorString(e)));
  }
  if (P->d.kernel == WAVE_KERNEL_TB2) {
    P->t2 = pick_t2();
    const size_t sm = P->t2.smem(P->d.pml_width);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, P->t2.fn);
    if ((e = cudaFuncSetAttribute(P->t2.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) != cudaSuccess)
      return bail(fail(WAVE_ERR_CUDA, "smem attribute (tb2): %s", cudaGetErrorString(e)));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, P->t2.fn, P->t2.nt, sm);
    if (occ < 1) return bail(fail(WAVE_ERR_CONFIG, "two-step kernel does not fit on an SM (w = %d)", P->d.pml_width));
    P->occ_t2 = occ;
    for (const void* f : {(const void*)k_source_at<float>, (const void*)k_source_at<double>, (const void*)k_advance}) cudaFuncGetAttributes(&fa, f);
  }
  *out = P;
  return WAVE_OK;
}

void wave_plan_destroy(wave_plan* P) {
  if (!P) return;
  drop_graphs(P);
  if (P->tab_d) cudaFree(P->tab_d);
  if (P->maps_g) cudaFree(P->maps_g);
  if (P->prog_d && (P->pair_dbg & 8) && P->pair_ok) {   // timing probe: dump the last launch's timeline
    const int n = P->pair_launch.nblk;
    std::vector<unsigned long long> h(6 * (size_t)n);
    cudaMemcpy(h.data(), P->prog_d + P->pair_launch.p.pair_dbg_off, h.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = fopen("pair_timeline.txt", "w")) {
      for (int i = 0; i < n; ++i)
        fprintf(f, "%d %llu %llu %llu %llu %llu %llu %llu\n", i, h[6 * i] >> 48, (h[6 * i] >> 32) & 0xffff,
                (h[6 * i] >> 16) & 0xffff, h[6 * i + 1], h[6 * i + 2], h[6 * i + 3], h[6 * i + 4] >> 32);
      fclose(f);
    }
  }
  if (P->pair_groups_d) cudaFree(P->pair_groups_d);
  if (P->mix_seq_d) cudaFree(P->mix_seq_d);
  if (P->prog_d) cudaFree(P->prog_d);
  if (P->dstep) cudaFree(P->dstep);
  if (P->stats_d) cudaFree(P->stats_d);
  if (P->ew_ctr) cudaFree(P->ew_ctr);
  if (P->ew_dbg) {
    unsigned long long h[6];
    cudaMemcpy(h, P->ew_dbg, sizeof h, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[ew] during interior: %llu units, %llu planes, %.3f us/plane; mop-up: %llu units, %llu planes, %.3f us/plane\n",
            h[4], h[1], h[1] ? h[0] * 1e-3 / h[1] : 0.0, h[5], h[3], h[3] ? h[2] * 1e-3 / h[3] : 0.0);
    cudaFree(P->ew_dbg);
  }
  if (P->ddone) cudaFree(P->ddone);
  if (P->inc_d) cudaFree(P->inc_d);
  if (P->wl_d) cudaFree(P->wl_d);
  if (P->side) cudaStreamDestroy(P->side);
  if (P->cap) cudaStreamDestroy(P->cap);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_join) cudaEventDestroy(P->ev_join);
  if (P->side2) cudaStreamDestroy(P->side2);
  if (P->ev_join2) cudaEventDestroy(P->ev_join2);
  delete P;
}

// Is the table division (div_table) bitwise the IEEE division for every B_d of
// this fp32 table?  Exhaustive device check (k_divcheck), cached per table.
static wave_status check_fastdiv(wave_plan* P, cudaStream_t s, bool* ok) {
  static std::mutex mu;
  static std::map<std::vector<float>, bool> cache;
  const int T = P->d.pml_width + 2;
  std::vector<float> key(P->tab_h.begin() + 2 * T, P->tab_h.begin() + 4 * T);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) { *ok = it->second; return WAVE_OK; }
  }
  unsigned* d = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned), s));
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned), s));
  k_divcheck<<<dim3(4 * 148, T), 256, 0, s>>>(static_cast<const float*>(P->tab_d), T, d);
  CK(cudaGetLastError());
  unsigned h = 1;
  CK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d, s));
  CK(cudaStreamSynchronize(s));
  *ok = h == 0;
  std::lock_guard<std::mutex> g(mu);
  cache[key] = *ok;
  return WAVE_OK;
}

static wave_status refresh_tables(wave_plan* P, cudaStream_t s) {
  make_constants(P->d, P->dt, &P->coef, &P->tab_h);
  make_constants64(P->d, P->dt, &P->coefd, &P->tab_hd);
  if (P->prec)
    CK(cudaMemcpyAsync(P->tab_d, P->tab_hd.data(), P->tab_hd.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  else
    CK(cudaMemcpyAsync(P->tab_d, P->tab_h.data(), P->tab_h.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));   // tab_h is pageable host memory
  P->fastdiv = false;
  if (P->prec == 0 && P->fastdiv_on) CKST(check_fastdiv(P, s, &P->fastdiv));
  CKST(build_launches(P));
  drop_graphs(P);
  return WAVE_OK;
}

// TMA descriptors of wavefield buffer b for every kernel that reads it
static wave_status encode_buffer(wave_plan* P, int b) {
  const uint64_t pb = P->L.pitch_x * P->esz, plb = pb * P->d.ny;
  const bool f64 = P->prec == 1;
  for (int ki = 0; ki < KI_N; ++ki) {
    const uint32_t TX = KTX(ki), CW = KCW(ki), TY = KTY(ki);
    if (ki == KI_SEAM) {
      // seam views: column 0 = x (nx - w - R) of row t - 1, t = 0..ny (ny + 1 seams)
      if (!P->L.seam || P->prec) continue;
      const int w = P->d.pml_width;
      float* sb = eo(P, P->buf[b], P->d.nx - w - R - P->L.pitch_x);
      CKST(encode3d(&P->maps[ki].u[b], sb, 2 * w + 2 * R, P->d.ny + 1, P->L.planes, pb, plb, TX + 2 * R, TY + 2 * R));
      CKST(encode3d(&P->maps[ki].up[b], sb, 2 * w + 2 * R, P->d.ny + 1, P->L.planes, pb, plb, CW, TY));
      continue;
    }
    // cluster kernels load the u window as (2R)-row boxes (multicast halves)
    const uint32_t UH = KCL(ki) > 1 ? 2 * R : TY + 2 * R;
    static const int xupromo = getenv("WAVE25_XWALL_UPROMO") ? atoi(getenv("WAVE25_XWALL_UPROMO")) : -1;  // A/B
    CKST(encode3d(&P->maps[ki].u[b], P->buf[b], P->d.nx, P->d.ny, P->L.planes, pb, plb, TX + 2 * R, UH, f64,
                  ki == KI_WALLX ? xupromo : -1, P->kt[ki].swz));
    CKST(encode3d(&P->maps[ki].up[b], P->buf[b], P->d.nx, P->d.ny, P->L.planes, pb, plb, CW, TY, f64,
                  centre_promo(P, ki, CW)));
  }
  if (P->d.kernel == WAVE_KERNEL_TB2) {
    const uint32_t TX = P->t2.tx, TY = P->t2.ty;
    CKST(encode3d(&P->t2maps.u[b], P->buf[b], P->d.nx, P->d.ny, P->L.planes, pb, plb, TX + 4 * R, TY + 4 * R));
    CKST(encode3d(&P->t2maps.up[b], P->buf[b], P->d.nx, P->d.ny, P->L.planes, pb, plb, TX + 2 * R, TY + 2 * R));
  }
  return WAVE_OK;
}

// device copy of the TMA descriptors (one per kernel kind and buffer, written
// once per bind): kernels can read them from global memory instead of from
// their parameter block (WAVE25_GMAPS)
static wave_status upload_maps(wave_plan* P) {
  if (!P->maps_g) CK(cudaMalloc(&P->maps_g, sizeof(P->maps)));
  CK(cudaMemcpy(P->maps_g, P->maps, sizeof(P->maps), cudaMemcpyHostToDevice));
  return WAVE_OK;
}

wave_status wave_plan_bind(wave_plan* P, float* u0, float* u1, float* vdt2, void* stream) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!u0 || !u1 || !vdt2 || u0 == u1) return fail(WAVE_ERR_CONFIG, "need two distinct wavefield buffers and vdt2");
  for (const void* p : {(const void*)u0, (const void*)u1, (const void*)vdt2})
    if (reinterpret_cast<uintptr_t>(p) % 128) return fail(WAVE_ERR_CONFIG, "buffers must be 128-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  P->base[0] = u0; P->base[1] = u1; P->base[2] = P->base[3] = nullptr; P->vdt2_base = vdt2;
  P->buf[0] = eo(P, u0, P->L.origin); P->buf[1] = eo(P, u1, P->L.origin); P->buf[2] = P->buf[3] = nullptr;
  P->vdt2 = eo(P, vdt2, P->L.origin);
  vdt2 = P->vdt2;
  P->aux = false;
  CK(cudaMemsetAsync(u0, 0, P->L.elems_u * P->esz, s));
  CK(cudaMemsetAsync(u1, 0, P->L.elems_u * P->esz, s));
  CK(cudaMemsetAsync(P->vdt2_base, 0, P->L.elems_vdt2 * P->esz, s));
  CK(cudaMemsetAsync(P->dstep, 0, sizeof(unsigned long long), s));
  const uint64_t pb = P->L.pitch_x * P->esz, plb = pb * P->d.ny;
  for (int ki = 0; ki < KI_N; ++ki) {
    if (ki == KI_SEAM) {
      if (!P->L.seam || P->prec) continue;
      const int w = P->d.pml_width;
      CKST(encode3d(&P->maps[ki].v, eo(P, vdt2, P->d.nx - w - R - P->L.pitch_x), 2 * w + 2 * R, P->d.ny + 1,
                    P->d.nz, pb, plb, KCW(ki), KTY(ki)));
      continue;
    }
    CKST(encode3d(&P->maps[ki].v, vdt2, P->d.nx, P->d.ny, P->d.nz, pb, plb, KCW(ki), KTY(ki), P->prec == 1,
                  centre_promo(P, ki, KCW(ki))));
  }
  if (P->d.kernel == WAVE_KERNEL_TB2) {
    CKST(encode3d(&P->t2maps.v1, vdt2, P->d.nx, P->d.ny, P->d.nz, pb, plb, P->t2.tx + 2 * R, P->t2.ty + 2 * R));
    CKST(encode3d(&P->t2maps.v2, vdt2, P->d.nx, P->d.ny, P->d.nz, pb, plb, P->t2.tx, P->t2.ty));
  }
  for (int b = 0; b < 2; ++b) CKST(encode_buffer(P, b));
  CKST(upload_maps(P));
  P->cur = 0;
  P->prv = 1;
  P->step = 0;
  P->bound = true;
  P->have_vel = false;
  if (P->dt > 0.f) CKST(refresh_tables(P, s));
  return WAVE_OK;
}

static wave_status rebuild_inc(wave_plan* P, cudaStream_t s) {
  if (!P->src_set || !P->src_local || !P->have_vel) return WAVE_OK;
  const int64_t k = P->sk - P->d.z_offset;
  const float* vsrc = eo(P, P->vdt2, (k * P->d.ny + P->sj) * P->L.pitch_x + P->si);
  const int64_t ns = (int64_t)P->wavelet.size();
  P->ninc = ns;
  if (ns == 0) return WAVE_OK;
  CK(cudaMemcpyAsync(P->wl_d, P->wavelet.data(), ns * sizeof(float), cudaMemcpyHostToDevice, s));
  const unsigned nb = (unsigned)std::min<int64_t>((ns + 255) / 256, 1024);
  if (P->prec)
    k_inc<double><<<nb, 256, 0, s>>>(static_cast<double*>(P->inc_d), P->wl_d, ns,
                                     reinterpret_cast<const double*>(vsrc));
  else
    k_inc<float><<<nb, 256, 0, s>>>(static_cast<float*>(P->inc_d), P->wl_d, ns, vsrc);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return WAVE_OK;
}

// stats over a padded-pitch field of fp32 (f64 = false) or fp64 elements
static wave_status field_stats(wave_plan* P, const float* base, int64_t rows, int positive, Stats* h,
                               cudaStream_t s, bool f64 = false) {
  Stats init{0u, 0x7f7fffffu, 0u, 0u};
  CK(cudaMemcpyAsync(P->stats_d, &init, sizeof init, cudaMemcpyHostToDevice, s));
  const int64_t n = rows * P->d.nx;
  (void)n;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(rows, 148 * 16));
  if (f64)
    k_stats<double><<<blocks, 256, 0, s>>>(reinterpret_cast<const double*>(base), P->L.pitch_x, (int)P->d.nx, rows,
                                           positive, P->stats_d);
  else
    k_stats<float><<<blocks, 256, 0, s>>>(base, P->L.pitch_x, (int)P->d.nx, rows, positive, P->stats_d);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h, P->stats_d, sizeof(Stats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return WAVE_OK;
}

wave_status wave_set_velocity(wave_plan* P, const float* vel, int32_t where, void* stream) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!P->bound) return fail(WAVE_ERR_STATE, "bind buffers before wave_set_velocity");
  if (!vel) return fail(WAVE_ERR_CONFIG, "vel is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rows = P->d.ny * P->d.nz;
  // V (fp32) goes into the vdt2 buffer itself (fp32 plans: converted in place)
  // or into a stream-ordered temporary (fp64 plans)
  float* vbuf = P->vdt2;
  if (P->prec) CK(cudaMallocAsync(reinterpret_cast<void**>(&vbuf), P->L.elems_vdt2 * sizeof(float), s));
  struct TmpFree {
    float* p; cudaStream_t s;
    ~TmpFree() { if (p) cudaFreeAsync(p, s); }
  } tmp_free{P->prec ? vbuf : nullptr, s};
  CK(cudaMemcpy2DAsync(vbuf, P->L.pitch_x * 4, vel, P->d.nx * 4, P->d.nx * 4, rows,
                       where == WAVE_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
  Stats st;
  CKST(field_stats(P, vbuf, rows, 1, &st, s));
  P->have_vel = false;
  if (st.bad) return fail(WAVE_ERR_CONFIG, "velocity must be finite and > 0 (%u bad values)", st.bad);
  float vmax;
  memcpy(&vmax, &st.max_bits, 4);
  float dt = P->d.dt;
  if (dt == 0.f) dt = (float)(0.4 * std::min(P->d.hx, std::min(P->d.hy, P->d.hz)) / (double)vmax);
  const double cn = courant_number(P->d, vmax, dt);
  if (cn > 1.0) return fail(WAVE_ERR_CONFIG, "dt = %g violates the Courant limit (ratio %.4f > 1)", dt, cn);
  P->dt = dt;
  if (P->prec)
    k_vdt2<double><<<(unsigned)std::min<int64_t>(rows, 148 * 16), 256, 0, s>>>(reinterpret_cast<double*>(P->vdt2), vbuf,
                                                                             P->L.pitch_x, (int)P->d.nx, rows,
                                           (double)dt);
  else
    k_vdt2<float><<<(unsigned)std::min<int64_t>(rows, 148 * 16), 256, 0, s>>>(P->vdt2, vbuf, P->L.pitch_x,
                                                                            (int)P->d.nx, rows, (double)dt);
  CK(cudaGetLastError());
  CKST(refresh_tables(P, s));
  P->have_vel = true;
  CKST(rebuild_inc(P, s));
  return WAVE_OK;
}

wave_status wave_set_source(wave_plan* P, int64_t i, int64_t j, int64_t k, const float* wl, int64_t ns,
                            void* stream) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!P->have_vel) return fail(WAVE_ERR_STATE, "set the velocity before the source");
  const int64_t w = P->d.pml_width;
  if (i < w || i >= P->d.nx - w || j < w || j >= P->d.ny - w || k < w || k >= P->d.nz_global - w)
    return fail(WAVE_ERR_CONFIG, "source (%lld,%lld,%lld) must lie inside the inner region", (long long)i,
                (long long)j, (long long)k);
  if (ns < 0 || (ns > 0 && !wl)) return fail(WAVE_ERR_CONFIG, "bad wavelet");
  cudaStream_t s = (cudaStream_t)stream;
  P->wavelet.assign(wl, wl + ns);
  if (P->inc_d) { cudaFree(P->inc_d); P->inc_d = nullptr; }
  if (P->wl_d) { cudaFree(P->wl_d); P->wl_d = nullptr; }
  if (ns > 0) {
    CK(cudaMalloc(&P->inc_d, ns * P->esz));
    CK(cudaMalloc(&P->wl_d, ns * sizeof(float)));
  }
  P->si = i; P->sj = j; P->sk = k;
  P->src_set = true;
  P->src_local = k >= P->d.z_offset && k < P->d.z_offset + P->d.nz;
  P->ninc = 0;
  drop_graphs(P);
  return rebuild_inc(P, s);
}

static wave_status ensure_peer_graph(wave_plan* P, int par);

wave_status wave_set_state(wave_plan* P, const float* uprev, const float* ucur, int32_t where, void* stream) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!P->bound) return fail(WAVE_ERR_STATE, "bind buffers first");
  cudaStream_t s = (cudaStream_t)stream;
  const cudaMemcpyKind kind = where == WAVE_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const float* src[4] = {ucur, uprev, nullptr, nullptr};
  for (int b = 0; b < 4; ++b) {
    if (!P->buf[b]) continue;
    CK(cudaMemsetAsync(P->base[b], 0, P->L.elems_u * P->esz, s));
    if (src[b])
      CK(cudaMemcpy2DAsync(eo(P, P->buf[b], R * P->L.pitch_x * P->d.ny), P->L.pitch_x * P->esz, src[b],
                           P->d.nx * P->esz, P->d.nx * P->esz, P->d.ny * P->d.nz, kind, s));
  }
  CK(cudaMemsetAsync(P->dstep, 0, sizeof(unsigned long long), s));
  // embedded-wall tickets re-armed too (they self-reset at every launch end; an
  // aborted launch would otherwise leave them mid-count)
  if (P->ew_ctr) CK(cudaMemsetAsync(P->ew_ctr, 0, 6 * sizeof(unsigned), s));
  if (P->have_peers) {
    // restart the step-flag protocol from 0 (collective: every rank of the
    // run re-initialises between two barriers) -- otherwise a
    // neighbour whose count matches the stale one could pass its wait and
    // store into ghost planes this call is about to zero
    CK(cudaMemsetAsync(P->ddone, 0, 2 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(P->peers.my_flags, 0, 2 * sizeof(uint64_t), s));
  }
  P->cur = 0;
  P->prv = 1;
  P->step = 0;
  // a velocity / source change since wave_set_peers dropped the peer graphs:
  // instantiate them now, not lazily while a neighbour's wait kernel spins
  if (P->have_peers && P->have_vel)
    for (int par = 0; par < 2; ++par) CKST(ensure_peer_graph(P, par));
  return WAVE_OK;
}

static wave_status ready(const wave_plan* P) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!P->bound) return fail(WAVE_ERR_STATE, "bind buffers first");
  if (!P->have_vel) return fail(WAVE_ERR_STATE, "set the velocity first");
  return WAVE_OK;
}

wave_status wave_step(wave_plan* P, int64_t nsteps, void* stream) {
  CKST(ready(P));
  if (nsteps < 0) return fail(WAVE_ERR_CONFIG, "nsteps < 0");
  if (P->d.nz != P->d.nz_global) return fail(WAVE_ERR_STATE, "multi-slab plan: use the split-step calls");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t left = nsteps;
  if (left >= 2 && pair_active(P)) {
    cudaGraphExec_t* g = &P->gexecP[P->cur * 4 + P->prv];
    if (!*g) CKST(capture(P, g, one_pair_l2, P->cur, P->prv));
    while (left >= 2) {                // in place: the state does not change
      CK(cudaGraphLaunch(*g, s));
      left -= 2;
      P->step += 2;
    }
  } else if (left >= 2 && tb2_active(P)) {
    while (left >= 2) {                // one graph per (cur, prv) state; a pair moves to (D, C)
      CKST(ensure_pair_graph(P, P->cur, P->prv));
      CK(cudaGraphLaunch(P->gexec2[P->cur * 4 + P->prv], s));
      int c, d;
      pair_targets(P->cur, P->prv, &c, &d);
      P->cur = d;
      P->prv = c;
      left -= 2;
      P->step += 2;
    }
  } else if (left >= 2) {
    CKST(ensure_graph(P, P->cur, P->prv));     // a 2-step graph returns to the same state
    while (left >= 2) {
      CK(cudaGraphLaunch(P->gexec[P->cur * 4 + P->prv], s));
      left -= 2;
      P->step += 2;
    }
  }
  if (left == 1) {
    CKST(enqueue_step(P, P->cur, P->prv, s));
    std::swap(P->cur, P->prv);
    P->step += 1;
  }
  return WAVE_OK;
}

wave_status wave_step_edges(wave_plan* P, void* stream) {
  CKST(ready(P));
  cudaStream_t s = (cudaStream_t)stream;
  CKST(enqueue_compute(P, 1, P->cur, P->prv, s));
  if (source_in(P, 1)) CKST(launch_source(P, P->prv, s));
  return WAVE_OK;
}

wave_status wave_step_interior(wave_plan* P, void* stream) {
  CKST(ready(P));
  cudaStream_t s = (cudaStream_t)stream;
  CKST(enqueue_compute(P, 2, P->cur, P->prv, s));
  if (source_in(P, 2)) CKST(launch_source(P, P->prv, s));
  return WAVE_OK;
}

wave_status wave_step_finish(wave_plan* P) {
  CKST(ready(P));
  std::swap(P->cur, P->prv);
  P->step += 1;
  return WAVE_OK;
}

wave_status wave_halo_views(const wave_plan* P, int32_t which, float** send_lo, float** send_hi,
                            float** recv_lo, float** recv_hi, int64_t* count) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  if (which != 0 && which != 1) return fail(WAVE_ERR_CONFIG, "which must be 0 or 1");
  const int64_t plane = P->L.pitch_x * P->d.ny, nz = P->d.nz;
  float* b = P->buf[which == 0 ? P->prv : P->cur];   // next (edges output) / current
  if (send_lo) *send_lo = eo(P, b, R * plane);
  if (send_hi) *send_hi = eo(P, b, nz * plane);
  if (recv_lo) *recv_lo = b;
  if (recv_hi) *recv_hi = eo(P, b, (nz + R) * plane);
  if (count) *count = R * plane;
  return WAVE_OK;
}

static wave_status enqueue_peer_step(wave_plan* P, int cur, cudaStream_t s);

static wave_status ensure_peer_graph(wave_plan* P, int par) {
  if (P->gexec_peer[par]) return WAVE_OK;
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(P->cap, cudaStreamCaptureModeThreadLocal));
  wave_status st = enqueue_peer_step(P, par, P->cap);
  if (st == WAVE_OK) st = enqueue_peer_step(P, 1 - par, P->cap);
  cudaError_t e = cudaStreamEndCapture(P->cap, &g);
  if (st != WAVE_OK) { if (g) cudaGraphDestroy(g); return st; }
  if (e != cudaSuccess) return fail(WAVE_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&P->gexec_peer[par], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(WAVE_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  return WAVE_OK;
}

// peer access from the current device to the device owning p (no-op if same)
static wave_status enable_peer_for(const void* p) {
  if (!p) return WAVE_OK;
  cudaPointerAttributes a{};
  CK(cudaPointerGetAttributes(&a, p));
  if (a.type != cudaMemoryTypeDevice) return fail(WAVE_ERR_CONFIG, "peer pointer is not device memory");
  int me = 0;
  CK(cudaGetDevice(&me));
  if (a.device == me || a.device < 0) return WAVE_OK;
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, me, a.device));
  if (!can) return fail(WAVE_ERR_CUDA, "device %d cannot access peer device %d", me, a.device);
  const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else if (e != cudaSuccess) return fail(WAVE_ERR_CUDA, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
  return WAVE_OK;
}

wave_status wave_ipc_export(const void* dptr, void* handle64, int64_t* offset) {
  if (!dptr || !handle64 || !offset) return fail(WAVE_ERR_CONFIG, "null argument");
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(WAVE_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  const CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr));
  if (r != CUDA_SUCCESS) return fail(WAVE_ERR_CUDA, "cuMemGetAddressRange failed (%d)", (int)r);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof h);
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dptr) - base);
  return WAVE_OK;
}

wave_status wave_ipc_import(const void* handle64, int64_t offset, void** base, void** dptr) {
  if (!handle64 || !base || !dptr || offset < 0) return fail(WAVE_ERR_CONFIG, "bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  void* b = nullptr;
  CK(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
  *base = b;
  *dptr = static_cast<char*>(b) + offset;
  return WAVE_OK;
}

wave_status wave_ipc_release(void* base) {
  if (!base) return WAVE_OK;
  CK(cudaIpcCloseMemHandle(base));
  return WAVE_OK;
}

wave_status wave_set_peers(wave_plan* P, const wave_peers* peers) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  drop_graphs(P);
  if (!peers) {
    P->have_peers = false;
    P->peers = wave_peers{};
    return WAVE_OK;
  }
  const bool lo = peers->lo_buf[0] && peers->lo_buf[1], hi = peers->hi_buf[0] && peers->hi_buf[1];
  if ((peers->lo_buf[0] != nullptr) != (peers->lo_buf[1] != nullptr) ||
      (peers->hi_buf[0] != nullptr) != (peers->hi_buf[1] != nullptr))
    return fail(WAVE_ERR_CONFIG, "give both buffers of a neighbour or none");
  if (!peers->my_flags || (lo && !peers->lo_flags) || (hi && !peers->hi_flags))
    return fail(WAVE_ERR_CONFIG, "flag words missing");
  if (lo && (P->d.z_offset == 0 || peers->lo_nz < R)) return fail(WAVE_ERR_CONFIG, "no lower neighbour at z_offset 0");
  if (hi && P->d.z_offset + P->d.nz >= P->d.nz_global) return fail(WAVE_ERR_CONFIG, "no upper neighbour at the top");
  if (P->d.kernel != WAVE_KERNEL_STREAM) return fail(WAVE_ERR_CONFIG, "peer stepping needs the stream kernels");
  for (const void* q : {(const void*)peers->lo_buf[0], (const void*)peers->lo_buf[1], (const void*)peers->hi_buf[0],
                        (const void*)peers->hi_buf[1], (const void*)peers->lo_flags, (const void*)peers->hi_flags})
    CKST(enable_peer_for(q));
  if (!P->ddone) CK(cudaMalloc(&P->ddone, 2 * sizeof(unsigned long long)));
  CK(cudaMemset(P->ddone, 0, 2 * sizeof(unsigned long long)));
  P->peers = *peers;
  // the neighbours' buffers are given as their allocations: element (0,0,-4)
  // is `origin` elements in (the neighbours have the same x geometry)
  for (int i = 0; i < 2; ++i) {
    if (P->peers.lo_buf[i]) P->peers.lo_buf[i] = eo(P, P->peers.lo_buf[i], P->L.origin);
    if (P->peers.hi_buf[i]) P->peers.hi_buf[i] = eo(P, P->peers.hi_buf[i], P->L.origin);
  }
  P->have_peers = true;
  // instantiate both parities' 2-step graphs now, before any peer-wait kernel
  // can be spinning on the device
  for (int par = 0; par < 2; ++par) CKST(ensure_peer_graph(P, par));
  return WAVE_OK;
}

static wave_status enqueue_peer_step(wave_plan* P, int cur, cudaStream_t s) {
  const bool lo = P->peers.lo_buf[0] != nullptr, hi = P->peers.hi_buf[0] != nullptr;
  using ull = unsigned long long;
  k_peer_wait<<<1, 1, 0, s>>>(reinterpret_cast<const ull*>(P->peers.my_flags), P->ddone, lo ? 1 : 0, hi ? 1 : 0,
                              P->ddone + 1, (ull)(P->peer_timeout_s * 1e9));
  CK(cudaGetLastError());
  P->remote = true;
  wave_status st = enqueue_compute(P, 0, cur, 1 - cur, s);
  if (st == WAVE_OK) st = launch_source(P, 1 - cur, s);
  P->remote = false;
  if (st != WAVE_OK) return st;
  k_peer_signal<<<1, 1, 0, s>>>(P->ddone, lo ? reinterpret_cast<ull*>(P->peers.lo_flags) : nullptr,
                                hi ? reinterpret_cast<ull*>(P->peers.hi_flags) : nullptr);
  CK(cudaGetLastError());
  return WAVE_OK;
}

wave_status wave_step_peer(wave_plan* P, int64_t nsteps, void* stream) {
  CKST(ready(P));
  if (!P->have_peers) return fail(WAVE_ERR_STATE, "call wave_set_peers first");
  if (nsteps < 0) return fail(WAVE_ERR_CONFIG, "nsteps < 0");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t left = nsteps;
  if (left >= 2) {
    const int par = P->cur;
    CKST(ensure_peer_graph(P, par));
    while (left >= 2) {
      CK(cudaGraphLaunch(P->gexec_peer[par], s));
      left -= 2;
      P->step += 2;
    }
  }
  if (left == 1) {
    CKST(enqueue_peer_step(P, P->cur, s));
    std::swap(P->cur, P->prv);
    P->step += 1;
  }
  return WAVE_OK;
}

wave_status wave_set_peer_timeout(wave_plan* P, double seconds) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!(seconds > 0.0) || seconds > 1e6) return fail(WAVE_ERR_CONFIG, "timeout must be in (0, 1e6] s");
  P->peer_timeout_s = seconds;
  drop_graphs(P);                 // the bound is baked into the captured wait kernels
  if (P->have_peers)
    for (int par = 0; par < 2; ++par) CKST(ensure_peer_graph(P, par));
  return WAVE_OK;
}

wave_status wave_peer_check(wave_plan* P, void* stream) {
  if (!P) return fail(WAVE_ERR_CONFIG, "plan is NULL");
  if (!P->ddone) return WAVE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long e = 0;
  CK(cudaMemcpyAsync(&e, P->ddone + 1, sizeof e, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (e)
    return fail(WAVE_ERR_PEER, "peer wait timed out after %.3g s (%s%s neighbour did not complete its step); "
                "the results of this run are invalid", P->peer_timeout_s, (e & 1) ? "lower" : "",
                (e & 3) == 3 ? " and upper" : (e & 2) ? "upper" : "");
  return WAVE_OK;
}

wave_status wave_push_halo(wave_plan* P, int32_t which, void* stream) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  if (!P->have_peers) return fail(WAVE_ERR_STATE, "call wave_set_peers first");
  if (which != 0 && which != 1) return fail(WAVE_ERR_CONFIG, "which must be 0 or 1");
  cudaStream_t s = (cudaStream_t)stream;
  const int bi = which == 1 ? P->cur : P->prv;
  const int64_t plane = P->L.pitch_x * P->d.ny, nz = P->d.nz, n4 = R * plane * (int64_t)P->esz / 16;
  const unsigned blocks = (unsigned)std::min<int64_t>((n4 + 255) / 256, 4 * 148);
  if (P->peers.lo_buf[bi]) {
    k_copy_planes<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(eo(P, P->buf[bi], R * plane)),
                                         reinterpret_cast<float4*>(eo(P, P->peers.lo_buf[bi], (P->peers.lo_nz + R) * plane)),
                                         n4);
    CK(cudaGetLastError());
  }
  if (P->peers.hi_buf[bi]) {
    k_copy_planes<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(eo(P, P->buf[bi], nz * plane)),
                                         reinterpret_cast<float4*>(P->peers.hi_buf[bi]), n4);
    CK(cudaGetLastError());
  }
  return WAVE_OK;
}

wave_status wave_read(const wave_plan* P, int32_t which, float* dst, int32_t where, void* stream) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  if (!dst || (which != 0 && which != 1)) return fail(WAVE_ERR_CONFIG, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const float* b = eo(P, P->buf[which == 0 ? P->cur : P->prv], R * P->L.pitch_x * P->d.ny);
  CK(cudaMemcpy2DAsync(dst, P->d.nx * P->esz, b, P->L.pitch_x * P->esz, P->d.nx * P->esz, P->d.ny * P->d.nz,
                       where == WAVE_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  if (where == WAVE_MEM_HOST) CK(cudaStreamSynchronize(s));
  return WAVE_OK;
}

wave_status wave_field_ptr(const wave_plan* P, int32_t which, float** out) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  if (!out || (which != 0 && which != 1)) return fail(WAVE_ERR_CONFIG, "bad arguments");
  *out = eo(P, P->buf[which == 0 ? P->cur : P->prv], R * P->L.pitch_x * P->d.ny);
  return WAVE_OK;
}

wave_status wave_check_finite(wave_plan* P, float* h_maxabs, void* stream) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  Stats st;
  CKST(field_stats(P, eo(P, P->buf[P->cur], R * P->L.pitch_x * P->d.ny), P->d.ny * P->d.nz, 0, &st,
                   (cudaStream_t)stream, P->prec == 1));
  float mx;
  memcpy(&mx, &st.max_bits, 4);
  if (h_maxabs) *h_maxabs = st.bad ? NAN : mx;
  if (st.bad)
    return fail(WAVE_ERR_UNSTABLE, "non-finite wavefield at step %lld (%u values)", (long long)P->step, st.bad);
  return WAVE_OK;
}

int64_t wave_step_index(const wave_plan* P) { return P ? P->step : -1; }

float wave_get_dt(const wave_plan* P) { return P ? P->dt : 0.f; }

// measurement kind of a kernel (the fused launch is the interior kind: it is
// the dominant kernel and covers every point)
static int kk_of(int ki) {
  return (ki == KI_FUSED || ki == KI_EW) ? WAVE_KK_INTERIOR
         : (ki == KI_WALLX_E || ki == KI_SEAM) ? WAVE_KK_XWALLS
         : ki == KI_WALLY_E ? WAVE_KK_YWALLS : ki;
}

static int64_t region_points(const std::vector<Launch>& Ls, int kind) {
  int64_t n = 0;
  for (const Launch& L : Ls)
    if (kk_of(L.ki) == kind)
      for (int r = 0; r < L.p.nreg; ++r) {
        const Region& g = L.p.reg[r];
        // (seams t = 0..ny: the right half of seam 0 and the left half of seam ny are not points)
        const int64_t rows = L.ki == KI_SEAM ? (int64_t)(g.y1 - g.y0 - 1) : (int64_t)(g.y1 - g.y0);
        n += (int64_t)(g.x1 - g.x0) * rows * (g.z1 - g.z0);
      }
  // embedded walls: the wall points are computed by the interior launch
  if (kind == WAVE_KK_INTERIOR)
    for (const Launch& L : Ls)
      if (L.ki == KI_EW)
        for (int r = 0; r < L.p.ew.nreg; ++r) {
          const Region& g = L.p.ew.reg[r];
          n += (int64_t)(g.x1 - g.x0) * (g.y1 - g.y0) * (g.z1 - g.z0);
        }
  return n;
}

wave_status wave_kernel_points(const wave_plan* P, int64_t* out) {
  if (!P || !out) return fail(WAVE_ERR_CONFIG, "bad arguments");
  for (int k = 0; k < WAVE_KK_N; ++k) out[k] = 0;
  if (tb2_active(P)) {
    const T2Params& q = P->t2p;
    out[WAVE_KK_INTERIOR] = (int64_t)(q.dx1 - q.dx0) * (q.dy1 - q.dy0) * q.nzl;
    for (int k = WAVE_KK_XWALLS; k <= WAVE_KK_YWALLS; ++k)
      out[k] = (region_points(P->wall_p1, k) + region_points(P->wall_p2, k)) / 2;
  } else {
    for (int k = 0; k < WAVE_KK_SOURCE; ++k) out[k] = region_points(P->launches[0], k);
  }
  out[WAVE_KK_SOURCE] = source_active(P) ? 1 : 0;
  return WAVE_OK;
}

wave_status wave_step_profiled(wave_plan* P, int64_t nsteps, void* stream, double* kernel_ms, int64_t* launches) {
  CKST(ready(P));
  if (nsteps < 0) return fail(WAVE_ERR_CONFIG, "nsteps < 0");
  if (P->d.nz != P->d.nz_global) return fail(WAVE_ERR_STATE, "multi-slab plan: use the split-step calls");
  if (P->d.kernel == WAVE_KERNEL_NAIVE) return fail(WAVE_ERR_STATE, "profiling needs the stream kernels");
  const bool pairl2 = pair_active(P);
  const bool pairs = tb2_active(P) || pairl2;
  if (pairs && nsteps % 2) return fail(WAVE_ERR_CONFIG, "two-step plans profile an even number of steps");
  cudaStream_t s = (cudaStream_t)stream;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  auto mk = [&](int kind, cudaStream_t st) -> wave_status {
    Rec r{kind, nullptr, nullptr};
    CK(cudaEventCreate(&r.a));
    CK(cudaEventCreate(&r.b));
    CK(cudaEventRecord(r.a, st));
    recs.push_back(r);
    return WAVE_OK;
  };
  const bool src = source_active(P);
  // every launch serialized on `stream` so every event pair brackets one kernel alone
  for (int64_t n = 0; n < nsteps; n += pairs ? 2 : 1) {
    const int cur = P->cur, prv = P->prv;
    if (pairl2) {
      CK(cudaMemsetAsync(P->prog_d, 0, P->prog_n * sizeof(unsigned), s));
      for (const Launch& L : P->launches[0])
        if (is_wall(L.ki)) {
          CKST(mk(kk_of(L.ki), s));
          CKST(launch_stream(P, L, cur, prv, P->buf[prv], s));
          CK(cudaEventRecord(recs.back().b, s));
        }
      if (src && source_in_frame(P, 0)) {
        CKST(mk(WAVE_KK_SOURCE, s));
        CKST(pair_wall_source(P, prv, 0, s));
        CK(cudaEventRecord(recs.back().b, s));
      }
      CKST(mk(WAVE_KK_INTERIOR, s));
      CKST(launch_pair_kernel(P, cur, prv, s));
      CK(cudaEventRecord(recs.back().b, s));
      for (const Launch& L : P->launches[0])
        if (is_wall(L.ki)) {
          CKST(mk(kk_of(L.ki), s));
          CKST(launch_stream(P, L, prv, cur, P->buf[cur], s));
          CK(cudaEventRecord(recs.back().b, s));
        }
      if (src && source_in_frame(P, 0)) {
        CKST(mk(WAVE_KK_SOURCE, s));
        CKST(pair_wall_source(P, cur, 1, s));
        CK(cudaEventRecord(recs.back().b, s));
      }
      if (src) {
        CKST(mk(WAVE_KK_SOURCE, s));
        k_advance<<<1, 1, 0, s>>>(P->dstep, 2);
        CK(cudaEventRecord(recs.back().b, s));
      }
      P->step += 2;
      continue;
    }
    if (pairs) {
      int c, d;
      pair_targets(cur, prv, &c, &d);
      for (const Launch& L : P->wall_p1) {
        CKST(mk(kk_of(L.ki), s));
        CKST(launch_stream(P, L, cur, prv, P->buf[c], s));
        CK(cudaEventRecord(recs.back().b, s));
      }
      if (src && source_in_frame(P, 8)) {
        CKST(mk(WAVE_KK_SOURCE, s));
        k_source_at<float><<<1, 1, 0, s>>>(P->buf[c], source_offset(P), static_cast<const float*>(P->inc_d), P->ninc,
                                    P->dstep, 0);
        CK(cudaEventRecord(recs.back().b, s));
      }
      for (const Launch& L : P->wall_p2) {
        CKST(mk(kk_of(L.ki), s));
        CKST(launch_stream(P, L, c, cur, P->buf[d], s));
        CK(cudaEventRecord(recs.back().b, s));
      }
      if (src && source_in_frame(P, 4)) {
        CKST(mk(WAVE_KK_SOURCE, s));
        k_source_at<float><<<1, 1, 0, s>>>(P->buf[d], source_offset(P), static_cast<const float*>(P->inc_d), P->ninc,
                                    P->dstep, 1);
        CK(cudaEventRecord(recs.back().b, s));
      }
      CKST(mk(WAVE_KK_INTERIOR, s));
      CKST(launch_t2(P, cur, prv, c, d, s));
      CK(cudaEventRecord(recs.back().b, s));
      if (src) {
        CKST(mk(WAVE_KK_SOURCE, s));
        k_advance<<<1, 1, 0, s>>>(P->dstep, 2);
        CK(cudaEventRecord(recs.back().b, s));
      }
      P->cur = d;
      P->prv = c;
      P->step += 2;
      continue;
    }
    for (const Launch& L : P->launches[0]) {
      CKST(mk(kk_of(L.ki), s));
      CKST(launch_stream(P, L, cur, prv, P->buf[prv], s));
      CK(cudaEventRecord(recs.back().b, s));
    }
    if (src) {
      CKST(mk(WAVE_KK_SOURCE, s));
      CKST(launch_source(P, prv, s));
      CK(cudaEventRecord(recs.back().b, s));
    }
    std::swap(P->cur, P->prv);
    P->step += 1;
  }
  CK(cudaStreamSynchronize(s));
  double ms[WAVE_KK_N] = {0, 0, 0, 0};
  int64_t cnt[WAVE_KK_N] = {0, 0, 0, 0};
  for (Rec& r : recs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.kind] += t;
    cnt[r.kind] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (int k = 0; k < WAVE_KK_N; ++k) {
    if (kernel_ms) kernel_ms[k] = ms[k];
    if (launches) launches[k] = cnt[k];
  }
  return WAVE_OK;
}

int32_t wave_launches_per_step(const wave_plan* P) {
  if (!P) return -1;
  int n = 0;
  const bool split = P->d.nz != P->d.nz_global;     // slab plans step via edges + interior
  if (P->d.kernel == WAVE_KERNEL_NAIVE) n = split ? 3 : 1;
  else n = split ? (int)(P->launches[1].size() + P->launches[2].size()) : (int)P->launches[0].size();
  if (source_active(P)) n += 1;
  return n;
}

int64_t wave_launches(const wave_plan* P, int64_t nsteps) {
  if (!P || nsteps < 0) return -1;
  if (P->have_peers)   // wave_step_peer: wait + all-plane compute launches + source + signal per step
    return nsteps * ((int64_t)P->launches[0].size() + (source_active(P) ? 1 : 0) + 2);
  const int64_t single = wave_launches_per_step(P);
  if (pair_active(P)) return (nsteps / 2) * pair_l2_launches(P) + (nsteps % 2) * single;
  if (!tb2_active(P)) return single * nsteps;
  return (nsteps / 2) * pair_launches(P) + (nsteps % 2) * single;
}

int32_t wave_steps_per_launch(const wave_plan* P) {
  if (!P) return -1;
  return (tb2_active(P) || pair_active(P)) ? 2 : 1;
}

wave_status wave_plan_bind_eta(wave_plan* P, float* eta_buf, void* stream) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "bind u0/u1/vdt2 first");
  if (!eta_buf || reinterpret_cast<uintptr_t>(eta_buf) % 128)
    return fail(WAVE_ERR_CONFIG, "eta buffer must be a 128-byte aligned device buffer");
  if (P->d.nz != P->d.nz_global) return fail(WAVE_ERR_CONFIG, "stored eta needs a single-slab plan");
  CK(cudaMemsetAsync(eta_buf, 0, P->L.elems_vdt2 * sizeof(float), (cudaStream_t)stream));
  P->eta_buf = eta_buf;
  P->eta_on = false;
  return WAVE_OK;
}

wave_status wave_set_eta(wave_plan* P, const float* eta, int32_t where, void* stream) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "plan not bound");
  cudaStream_t s = (cudaStream_t)stream;
  if (!eta) {                               // back to the eta_max (d/w)^2 profile
    P->eta_on = false;
  } else {
    if (!P->eta_buf) return fail(WAVE_ERR_STATE, "call wave_plan_bind_eta first");
    const int64_t rows = P->d.ny * P->d.nz;
    CK(cudaMemcpy2DAsync(P->eta_buf, P->L.pitch_x * 4, eta, P->d.nx * 4, P->d.nx * 4, rows,
                         where == WAVE_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    Stats st;
    CKST(field_stats(P, P->eta_buf, rows, 2, &st, s));
    if (st.bad) {
      P->eta_on = false;
      return fail(WAVE_ERR_CONFIG, "eta must be finite and >= 0 (%u bad values)", st.bad);
    }
    P->eta_on = true;
  }
  if (P->dt > 0.f) CKST(build_launches(P));
  drop_graphs(P);
  return WAVE_OK;
}

wave_status wave_plan_bind_aux(wave_plan* P, float* u2, float* u3, void* stream) {
  if (!P || !P->bound) return fail(WAVE_ERR_STATE, "bind u0/u1/vdt2 first");
  if (!u2 || !u3 || u2 == u3 || u2 == P->base[0] || u2 == P->base[1] || u3 == P->base[0] || u3 == P->base[1])
    return fail(WAVE_ERR_CONFIG, "need two more distinct wavefield buffers");
  for (const void* p : {(const void*)u2, (const void*)u3})
    if (reinterpret_cast<uintptr_t>(p) % 128) return fail(WAVE_ERR_CONFIG, "buffers must be 128-byte aligned");
  if (P->d.kernel != WAVE_KERNEL_TB2) return fail(WAVE_ERR_CONFIG, "aux buffers are for WAVE_KERNEL_TB2 plans");
  cudaStream_t s = (cudaStream_t)stream;
  P->base[2] = u2;
  P->base[3] = u3;
  P->buf[2] = eo(P, u2, P->L.origin);
  P->buf[3] = eo(P, u3, P->L.origin);
  CK(cudaMemsetAsync(u2, 0, P->L.elems_u * sizeof(float), s));
  CK(cudaMemsetAsync(u3, 0, P->L.elems_u * sizeof(float), s));
  for (int b = 2; b < 4; ++b) CKST(encode_buffer(P, b));
  CKST(upload_maps(P));
  P->aux = true;
  drop_graphs(P);
  return WAVE_OK;
}

}  // extern "C"
