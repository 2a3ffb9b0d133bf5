// Load-time generated pass kernels (see jit.h and DESIGN.md §5).
//
// A pass of the compiled program reads every amplitude of the (shard) state once, applies the
// pass's ops in registers and writes it back once (2S bytes, the algorithmic minimum per pass).
// The ahead-of-time pass kernel interprets the op list at run time; these kernels instead bake
// the op list into straight-line code, so that
//   * complex64 butterflies run on packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100a):
//     y = a x1 (FMUL2 + FFMA2 with the swapped-operand modifier), x0 +- y (FADD2) = 2 instructions
//     per amplitude for a butterfly on a register slot;
//   * an unconditional X on a register slot is a compile-time renaming (no instruction);
//   * the CZ sign of an absorbed E is a compile-time add/sub swap when its slot is a register bit,
//     a per-thread coefficient sign when it is a lane, group-base or rank bit;
//   * no register reconciliation at op-dispatch merge points (there are none).
// Layout per warp unit (identical to the AOT kernel, so both agree on every index): a warp moves a
// 512 B contiguous segment per vector (complex64: float4 = 2 amplitudes per lane, slot 0 in the
// vector, slots 1..5 on lane bits; complex128: double2, slots 0..4 on lane bits); every thread
// holds the 2^KHI segments that differ in the pass's group slots, UNR units per loop trip.
#include "jit.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <functional>
#include <type_traits>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cctype>
#include <array>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

namespace owqs {

namespace {
#include "jit_prelude.inc"  // kPreludeInternal (owqs_internal.h), kPreludeCommon (device_common.cuh)

// Device helpers used only by the generated kernels: packed fp32x2 arithmetic (PTX ISA f32x2,
// sm_100a) on a complex64 amplitude held as one 64-bit register pair (re = low, im = high).
const char* kHelpers = R"OWQS(
typedef unsigned long long u64;
#define OWQS_SIGN2 0x8000000080000000ull
static __device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
static __device__ __forceinline__ float lo(u64 r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a; }
static __device__ __forceinline__ float hi(u64 r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return b; }
static __device__ __forceinline__ u64 swp(u64 x) { return pk(hi(x), lo(x)); }
static __device__ __forceinline__ u64 bc(float a) { return pk(a, a); }
static __device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
static __device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
static __device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
static __device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
static __device__ __forceinline__ u64 shfl2(u64 x, int m) { return pk(__shfl_xor_sync(0xffffffffu, lo(x), m), __shfl_xor_sync(0xffffffffu, hi(x), m)); }
static __device__ __forceinline__ u64 neg2(u64 x) { return pk(-lo(x), -hi(x)); }
static __device__ __forceinline__ u64 flip2(u64 x, unsigned f) { return x ^ (((u64)f << 63) | ((u64)f << 31)); }
static __device__ __forceinline__ double fld(double x, unsigned f) { return __longlong_as_double(__double_as_longlong(x) ^ ((unsigned long long)f << 63)); }
)OWQS";

// FNV-1a 64
uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::string hex64(uint64_t v) {
  char b[17];
  snprintf(b, sizeof b, "%016llx", (unsigned long long)v);
  return b;
}

enum SlotKind { SK_REG, SK_LANE, SK_WARP, SK_BASE, SK_RANK };

// ---- engine 2: the CTA tile ---------------------------------------------------------------------
// A CTA (8 warps) owns a tile of 2^TB amplitudes: tile bits t0..t(SB-1) = the warp segment's slots
// (512 B: 64 complex64 / 32 complex128 amplitudes), the next 7 = the pass's group slots ascending
// (padded with untouched base slots); TB = 13 (complex64) / 12 (complex128). A layout maps the tile
// bits onto (register position bit k: R[k], lane bit j: Lb[j], warp bit j: Wb[j]). complex64: R[0] =
// t0 always, so every thread holds slot-0 neighbours as float4 pairs, 32 amplitudes per thread;
// complex128: one double2 per amplitude, 16 per thread. Layouts whose lanes are the segment's lane
// slots (t1..t5 / t0..t4) and whose other register bits are group bits ("A-type") are the ones
// global loads and stores use (coalesced 512 B per warp instruction); the others are reached
// through the shared-memory tile. 16 B unit of tile index t: u(t) = v + (v >> 3) + (v >> 6) + (v >> 9),
// v = t >> 1 (complex64 pairs) or t (complex128). u is injective and additive over disjoint bit sets
// (per-thread base + per-register immediate), and a tile bit lands in bank group 2^(class mod 3)
// (mod 8), class = k - 1 (complex64) or k: a quarter-warp is conflict-free when lane bits 0, 1, 2
// carry tile bits of the three classes.
struct CLayout {
  int R[6];   // R[0] = t0; R[1..RB-1] used
  int Lb[5];
  int Wb[3];  // Wb[0..WB-1] used
};
// Tile geometry: RB register bits per thread (2^RB amplitudes) + 5 lane bits + WB warp bits = 13.
// RB = 5, WB = 3: 8-warp CTAs, 32 amplitudes per thread (default); RB = 6, WB = 2: 4-warp CTAs,
// 64 amplitudes per thread (OWQS_TILE_RB=6).
struct TileGeom {
  int rb, wb;
};
// group slots of a complex64 tile: 6 (default: 12-bit tiles, 4-warp CTAs, 4 CTAs per SM) or
// OWQS_TILE_G = 7 (13-bit tiles, 8-warp CTAs, 2 per SM) / 5 (2-warp CTAs, 8 per SM). Measured on C3:
// 43.5 / 44.6 / 47.1 ms -- 6 needs 38 passes instead of 35 but four independent CTAs per SM overlap
// their load / compute / transpose phases better. complex128 keeps KTILE.
inline int tile_g(int prec) {
  static const int g = [] {
    const char* e = getenv("OWQS_TILE_G");
    return (e && atoi(e) >= 5 && atoi(e) <= KTILE) ? atoi(e) : 6;
  }();
  static const int g128 = [] {  // complex128: 6 (11-bit tiles, 4-warp CTAs, 4 per SM: C3 94.9 ms)
    const char* e = getenv("OWQS_TILE_G128");  // 7 (8-warp CTAs): 96.1 ms, 5: 97.3 ms
    return (e && atoi(e) >= 5 && atoi(e) <= KTILE) ? atoi(e) : 6;
  }();
  return prec == 0 ? g : g128;
}
inline TileGeom tile_geom() {
  static const TileGeom g = [] {
    const char* e = getenv("OWQS_TILE_RB");
    int rb = (e && atoi(e) >= 4 && atoi(e) <= 6) ? atoi(e) : 5;
    if (1 + tile_g(0) - rb < 1) rb = 5;  // at least one warp bit
    return TileGeom{rb, 1 + tile_g(0) - rb};  // 6 + G tile bits = RB + 5 lane bits + WB
  }();
  return g;
}
inline int tile_bits(int prec) { return (prec == 0 ? 6 : 5) + tile_g(prec); }
// 16 B unit of tile index t: v = t >> 1 (complex64 pairs) or t, XOR-swizzled in its low 3 bits by
// the higher ones: u = v ^ ((v >> 3 ^ v >> 6 ^ v >> 9) & 7). u is a bijection, linear over GF(2)
// (per-thread base XOR per-register constant), exactly 64 KB for both precisions, and tile bit k
// lands in bank group 2^(class mod 3) -- the same conflict-freedom rule as a padded layout
inline int umap_p(int t, int prec) {
  const int v = prec == 0 ? t >> 1 : t;
  return v ^ (((v >> 3) ^ (v >> 6) ^ (v >> 9)) & 7);
}
constexpr int kTileSmem = 16 * 4096;

struct Gen {
  const StepDesc& d;
  const int prec;
  const bool tile;  // engine 2
  const int SB, EPV;
  int KHI, G, UNR, P;
  int RB = 5, WB = 3;  // tile engine geometry
  int TB = 13;         // tile bits
  int FB = 1;          // first register-selectable tile bit (complex64: t0 is fixed in R[0])
  int LS = 1;          // first segment lane slot of global IO layouts (complex64: t1, t0 pairs float4)
  bool t0free = false; // complex64, OWQS_T0_FREE: phases may leave t0 out of the registers
  int NSEL = 4;        // register tile bits a phase selects
  // per-kernel shared-memory map (choose_bank_classes): uval[k] = 16 B unit of tile bit k alone
  bool ucustom = false;
  int uval[16] = {}, ucls[16] = {};
  // byte offset of tile index t in the shared-memory tile: 16 B unit, plus 8 B for t0 (complex64)
  int addrb(int t) const { return 16 * umap(t) ^ ((prec == 0 && (t & 1)) ? 8 : 0); }
  int umap(int t) const {
    if (!ucustom) return umap_p(t, prec);
    int u = 0;
    for (int k = 0; k < 16; ++k)
      if ((t >> k) & 1) u ^= uval[k];
    return u;
  }
  int bclass(int k) const { return ucustom ? ucls[k] : (prec == 0 ? (k - 1) % 3 : k % 3); }
  // Bank classes chosen for this kernel: a 3-colouring of the tile bits (t1.. for complex64, t0..
  // for complex128) such that every used layout's 5 lane bits hold all three classes, so its lane
  // bits 0..2 can take one each (quarter-warp 16 B accesses conflict-free). Branch and bound over
  // 3^12 colourings (fewest non-rainbow lane sets; the default colouring first). Then the map:
  // u bit c (c < 3) = XOR of the v-bits of class c, u bits 3.. = the non-pivot v-bits in order --
  // a GF(2) bijection of the 12 v-bits (v = t >> 1 complex64, t complex128) onto 64 KB.
  void choose_bank_classes(const std::vector<int>& used) {
    const int lo = LS, nb = TB - LS;  // complex64: t0 is the 8 B half of a unit, not a bank bit
    std::vector<uint32_t> edges;
    for (int l : used) {
      uint32_t m = 0;
      for (int j = 0; j < 5; ++j) m |= 1u << lays[l].Lb[j];
      if (prec == 0) m &= ~1u;
      if (std::find(edges.begin(), edges.end(), m) == edges.end()) edges.push_back(m);
    }
    int cls[16], best[16], best_bad = 1 << 30;
    for (int k = 0; k < 16; ++k) cls[k] = best[k] = -1;
    auto bad_edges = [&](int upto) {  // edges fully coloured among bits < upto that miss a class
      int bad = 0;
      for (uint32_t m : edges) {
        if (m >> upto) continue;
        int seen = 0;
        for (int k = lo; k < upto; ++k)
          if ((m >> k) & 1) seen |= 1 << cls[k];
        bad += seen != 7;
      }
      return bad;
    };
    long long budget = 2000000;
    std::function<void(int)> dfs = [&](int k) {
      if (--budget < 0) return;
      const int bad = bad_edges(k);
      if (bad >= best_bad) return;
      if (k == TB) {
        best_bad = bad;
        std::copy(cls, cls + 16, best);
        return;
      }
      const int def = (k - lo) % 3;  // default colouring tried first
      for (int c0 = 0; c0 < 3 && best_bad > 0; ++c0) {
        cls[k] = (def + c0) % 3;
        dfs(k + 1);
      }
      cls[k] = -1;
    };
    dfs(lo);
    if (best_bad == 1 << 30) return;
    int pivot[3] = {-1, -1, -1};
    for (int k = lo; k < TB; ++k)
      if (pivot[best[k]] < 0) pivot[best[k]] = k;
    if (pivot[0] < 0 || pivot[1] < 0 || pivot[2] < 0) return;
    ucustom = true;
    int hi = 3;
    for (int k = 0; k < 16; ++k) uval[k] = 0, ucls[k] = 0;
    for (int k = lo; k < TB; ++k) {
      ucls[k] = best[k];
      uval[k] = 1 << best[k];
      if (k != pivot[best[k]]) uval[k] |= 1 << hi++;
    }
    (void)nb;
    // lane order: one bit of each class on lane bits 0..2 where the set allows; t0 (complex64, not
    // a register bit: 8 B accesses, half-warp wavefronts) on lane bit 3
    for (int l : used) {
      CLayout& L = lays[l];
      int order[5], n = 0;
      bool taken[5] = {};
      for (int c = 0; c < 3; ++c)
        for (int j = 0; j < 5; ++j)
          if (!taken[j] && L.Lb[j] >= lo && ucls[L.Lb[j]] == c) {
            taken[j] = true;
            order[n++] = L.Lb[j];
            break;
          }
      if (prec == 0)
        for (int j = 0; j < 5; ++j)
          if (!taken[j] && L.Lb[j] == 0) {
            while (n < 3) {  // fewer than 3 classes: fill before t0 (conflicts, still correct)
              int k = 0;
              while (k < 5 && (taken[k] || L.Lb[k] == 0)) ++k;
              if (k == 5) break;
              taken[k] = true;
              order[n++] = L.Lb[k];
            }
            taken[j] = true;
            order[n++] = 0;
          }
      for (int j = 0; j < 5; ++j)
        if (!taken[j]) order[n++] = L.Lb[j];
      for (int j = 0; j < 5; ++j) L.Lb[j] = order[j];
    }
  }
  int gs[KMAX_HI];  // group slots (engine 2: padded to KTILE)
  std::vector<CLayout> lays;  // engine 2 layouts used by this kernel
  int lay = 0;                // engine 2: current layout index
  std::ostringstream o;
  std::vector<int> perm;  // logical register position -> variable id
  struct Pend {
    int a, b, idx;
    bool cond;
  };
  std::vector<Pend> pend;
  std::string error;

  // coefficient source of a tile kernel: "cp." = the kernel's by-value PassCoef parameter (constant
  // bank: uniform-register FFMA2 / DFMA operands, written into the graph node by decide_kernel or by
  // the host for EOWQS), "pc->" = the PassCoef decide_kernel wrote to global memory (registers)
  std::string PC = "pc->";
  int coef_src = 0;  // 0 pointer, 1 by-value parameter, 2 module __constant__ (jit.h)
  Gen(const StepDesc& dd, int pr, bool use_tile, bool free_t0 = false, int csrc = 0)
      : d(dd), prec(pr), tile(use_tile), SB(pr == 0 ? 6 : 5), EPV(pr == 0 ? 2 : 1) {
    coef_src = use_tile ? csrc : 0;
    if (coef_src == 1) PC = "cp.";
    if (coef_src == 2) PC = "OWQS_KNAME_cp.";
    if (tile) {
      KHI = tile_g(pr);
      UNR = 1;
      int n = 0;
      for (int j = 0; j < d.nb_hi; ++j) gs[n++] = d.bhi[j];
      for (int s = SB; n < KHI && s < d.width; ++s) {
        bool used = false;
        for (int j = 0; j < n; ++j) used = used || gs[j] == s;
        if (!used) gs[n++] = s;
      }
      if (n < KHI) error = "tile engine needs width >= SB + group slots";
      std::sort(gs, gs + KHI);
      TB = tile_bits(prec);
      if (prec == 0) {
        RB = tile_geom().rb;
        WB = tile_geom().wb;
        t0free = free_t0 && RB <= 5;  // a phase holds at most 5 selected bits (Phase::S)
        FB = t0free ? 0 : 1;
        LS = 1;
        NSEL = t0free ? RB : RB - 1;
      } else {
        RB = 4;
        WB = tile_g(1) - 4;  // 5 + G tile bits = 4 register + 5 lane + WB warp bits
        FB = 0;
        LS = 0;
        NSEL = 4;
      }
      P = 1 << RB;
    } else {
      KHI = d.nb_hi;
      UNR = jit_unr_of(KHI);
      for (int j = 0; j < KHI; ++j) gs[j] = d.bhi[j];
      P = (UNR << KHI) * EPV;
    }
    G = 1 << KHI;
    for (int p = 0; p < P; ++p) perm.push_back(p);
  }

  int tilebit(int s) const {
    if (s < SB) return s;
    for (int j = 0; j < KHI; ++j)
      if (gs[j] == s) return SB + j;
    return -1;
  }
  // kind of slot s in layout l (engine 2) / the fixed direct layout (engine 1); *bit = position
  // mask (REG), lane bit (LANE), warp bit (WARP), bit of gb (BASE) or rank bit (RANK)
  int kind_l(int s, int l, int* bit) const {
    if (s >= d.width) {
      *bit = s - d.width;
      return SK_RANK;
    }
    const int tb = tilebit(s);
    if (tb < 0) {
      *bit = s - SB;
      return SK_BASE;
    }
    if (tile) {
      const CLayout& L = lays[l];
      for (int k = 0; k < RB; ++k)
        if (L.R[k] == tb) {
          *bit = 1 << k;
          return SK_REG;
        }
      for (int j = 0; j < 5; ++j)
        if (L.Lb[j] == tb) {
          *bit = j;
          return SK_LANE;
        }
      for (int j = 0; j < WB; ++j)
        if (L.Wb[j] == tb) {
          *bit = j;
          return SK_WARP;
        }
      return SK_BASE;  // unreachable
    }
    if (EPV == 2 && s == 0) {
      *bit = 1;
      return SK_REG;
    }
    if (s < SB) {
      *bit = s - (EPV == 2 ? 1 : 0);
      return SK_LANE;
    }
    *bit = EPV << (tb - SB);
    return SK_REG;
  }
  int kind(int s, int* bit) const { return kind_l(s, lay, bit); }
  bool is_reg(int s) const {
    int b;
    return kind(s, &b) == SK_REG;
  }
  int pbit(int s) const {
    int b;
    kind(s, &b);
    return b;
  }
  int regval(int s, int p) const { return (p & pbit(s)) ? 1 : 0; }
  int unit_of(int p) const { return tile ? 0 : p / (G * EPV); }

  std::string X(int p) const { return "x" + std::to_string(perm[p]); }
  std::string XR(int p) const { return "xr" + std::to_string(perm[p]); }
  std::string XI(int p) const { return "xi" + std::to_string(perm[p]); }

  // parity of the runtime (non-register) bits of slot mask m for unit u; "" if none
  std::string rt_parity(uint64_t m, int u) const {
    uint32_t L = 0, R = 0, W = 0;
    uint64_t B = 0;
    for (int s = 0; s < 64; ++s) {
      if (!((m >> s) & 1)) continue;
      int b;
      int k = kind(s, &b);
      if (k == SK_LANE) L |= 1u << b;
      if (k == SK_WARP) W |= 1u << b;
      if (k == SK_BASE) B |= 1ull << b;
      if (k == SK_RANK) R |= 1u << b;
    }
    std::vector<std::string> t;
    if (L) t.push_back("__popc(lane & " + std::to_string(L) + "u)");
    if (W) t.push_back("__popc(warp & " + std::to_string(W) + "u)");
    if (B) t.push_back("__popcll(gb" + std::to_string(u) + " & " + std::to_string(B) + "ull)");
    if (R) t.push_back("__popc(rk & " + std::to_string(R) + "u)");
    if (t.empty()) return "";
    std::string e = "((";
    for (size_t i = 0; i < t.size(); ++i) e += (i ? " + " : "") + t[i];
    return e + ") & 1u)";
  }
  // static parity of the register bits of mask m at position p
  int st_parity(uint64_t m, int p) const {
    int r = 0;
    for (int s = 0; s < 64; ++s)
      if (((m >> s) & 1) && is_reg(s)) r ^= regval(s, p);
    return r;
  }
  // runtime value (0/1) of bit s for unit u (s not a register slot)
  std::string rt_bit(int s, int u) const {
    int b;
    int k = kind(s, &b);
    if (k == SK_LANE) return "((unsigned)(lane >> " + std::to_string(b) + ") & 1u)";
    if (k == SK_WARP) return "((unsigned)(warp >> " + std::to_string(b) + ") & 1u)";
    if (k == SK_BASE) return "((unsigned)(gb" + std::to_string(u) + " >> " + std::to_string(b) + ") & 1u)";
    return "((rk >> " + std::to_string(b) + ") & 1u)";
  }
  std::string cond_expr(int i) const { return (tile ? PC + "cond[" : std::string("sh.cond[")) + std::to_string(i) + "]"; }

  // own-tile L2 bulk prefetch before griddepcontrol.wait: off by default since the kernels stopped
  // being instruction-fetch bound (ptxas -O1, tile planning): C3 34.48 -> 33.96 ms without it
  // (OWQS_PDL_PREFETCH=1: on)
  static bool pdl_prefetch() {
    static const bool v = getenv("OWQS_PDL_PREFETCH") && atoi(getenv("OWQS_PDL_PREFETCH")) != 0;
    return v;
  }
  static int prefetch_distance() {
    // 13-bit tiles (2 CTAs per SM): one wave ahead, 148 x 2, measured C3 49.8 -> 49.3 ms, C3W 219 ->
    // 213 ms. 12-bit tiles (4 CTAs per SM, default): off -- the extra resident CTAs already hide the
    // load latency and the prefetch costs issue slots (C3 43.4 -> 42.8 ms, C3E 42.8 -> 41.2 ms)
    static const int v = getenv("OWQS_PREFETCH") ? atoi(getenv("OWQS_PREFETCH"))
                                                 : (tile_g(0) == KTILE ? 148 * tile_minb_for(0) : 0);
    return v;
  }
  void bfly(int i, int bi) {
    const Op& op = d.ops[i];
    const int a = op.a;
    const uint64_t am = d.absorb[bi];
    int lb;
    const int ka = kind(a, &lb);
    o << "    {  // op " << i << ": butterfly " << bi << " on slot " << a << (ka == SK_REG ? " (register)" : " (lane)")
      << "\n";
    // the pass's normalisation scale folded into its first butterfly (tile engine): out = k x0 +- (k a) x1
    // costs the same 4 packed ops as x0 +- a x1, and saves the separate multiply of every amplitude
    const bool fold = tile && scale_pending;
    if (fold) scale_pending = false;
    if (fold && prec == 0)
      o << "      const float ar = " << PC << "ar[" << bi << "] * sck; const u64 cB = mul2(" << PC << "B[" << bi << "], bc(sck));  // scale folded\n";
    else if (fold)
      o << "      const double ar = " << PC << "ard[" << bi << "] * sck, ai = " << PC << "aid[" << bi << "] * sck;  // scale folded\n";
    else if (tile && prec == 0)
      o << "      const float ar = " << PC << "ar[" << bi << "]; const u64 cB = " << PC << "B[" << bi << "];\n";
    else if (tile)
      o << "      const double ar = " << PC << "ard[" << bi << "], ai = " << PC << "aid[" << bi << "];\n";
    else if (prec == 0)
      o << "      const float ar = s_ar[" << bi << "]; const u64 cB = s_B[" << bi << "];\n";
    else
      o << "      const double ar = s_ar[" << bi << "], ai = s_ai[" << bi << "];\n";
    // coefficient with the runtime part of the absorbed-CZ sign, per unit
    for (int u = 0; u < UNR; ++u) {
      std::string t = rt_parity(am, u);
      if (t.empty()) {
        if (prec == 0)
          o << "      const float ar" << u << " = ar; const u64 B" << u << " = cB;\n";
        else
          o << "      const double ar" << u << " = ar, ai" << u << " = ai;\n";
      } else {
        o << "      const unsigned t" << u << " = " << t << ";\n";
        if (prec == 0)
          o << "      const float ar" << u << " = t" << u << " ? -ar : ar; const u64 B" << u << " = t" << u
            << " ? (cB ^ OWQS_SIGN2) : cB;\n";
        else
          o << "      const double ar" << u << " = t" << u << " ? -ar : ar, ai" << u << " = t" << u << " ? -ai : ai;\n";
      }
    }
    if (ka == SK_REG) {
      const int pb = lb;
      for (int p = 0; p < P; ++p) {
        if (p & pb) continue;
        const int p1 = p | pb, u = unit_of(p);
        const int s = st_parity(am, p);
        if (prec == 0 && fold) {
          o << "      { const u64 y = fma2(B" << u << ", swp(" << X(p1) << "), mul2(bc(ar" << u << "), " << X(p1)
            << ")); const u64 t = " << X(p) << "; " << X(p) << " = fma2(bc(sck), t, " << (s ? "neg2(y)" : "y") << "); "
            << X(p1) << " = fma2(bc(sck), t, " << (s ? "y" : "neg2(y)") << "); }\n";
        } else if (prec == 0) {
          // w = x0 + a x1 (2 FMA), the other row 2 x0 - w (1 FMA): 3 packed ops per pair instead of 4
          const std::string w = s ? X(p1) : X(p), r = s ? X(p) : X(p1);
          o << "      { const u64 t = " << X(p) << "; const u64 w = fma2(bc(ar" << u << "), " << X(p1) << ", fma2(B" << u
            << ", swp(" << X(p1) << "), t)); " << r << " = fma2(bc(2.f), t, neg2(w)); " << w << " = w; }\n";
        } else if (fold) {
          const std::string u_ = std::to_string(u);
          o << "      { const double yr = ar" << u_ << " * " << XR(p1) << " - ai" << u_ << " * " << XI(p1)
            << ", yi = ar" << u_ << " * " << XI(p1) << " + ai" << u_ << " * " << XR(p1) << "; const double tr = "
            << XR(p) << ", ti = " << XI(p) << "; " << XR(p) << " = fma(sck, tr, " << (s ? "-" : "") << "yr); " << XI(p)
            << " = fma(sck, ti, " << (s ? "-" : "") << "yi); " << XR(p1) << " = fma(sck, tr, " << (s ? "" : "-")
            << "yr); " << XI(p1) << " = fma(sck, ti, " << (s ? "" : "-") << "yi); }\n";
        } else {
          // w = x0 + a x1 (4 DFMA), the other row 2 x0 - w (2 DFMA)
          const std::string u_ = std::to_string(u);
          const std::string wr = s ? XR(p1) : XR(p), wi = s ? XI(p1) : XI(p), rr = s ? XR(p) : XR(p1),
                            ri = s ? XI(p) : XI(p1);
          o << "      { const double tr = " << XR(p) << ", ti = " << XI(p) << "; const double wr = fma(ar" << u_ << ", "
            << XR(p1) << ", fma(-ai" << u_ << ", " << XI(p1) << ", tr)), wi = fma(ar" << u_ << ", " << XI(p1) << ", fma(ai"
            << u_ << ", " << XR(p1) << ", ti)); " << rr << " = fma(2.0, tr, -wr); " << ri << " = fma(2.0, ti, -wi); "
            << wr << " = wr; " << wi << " = wi; }\n";
        }
      }
    } else if (ka == SK_LANE) {
      // lower lane holds x0, upper x1. Each lane sends y = c x (c = 1 lower, +-a upper) and keeps
      // out = r + sg y (sg = +1 lower, -1 upper): lower x0 + a x1, upper x0 - a x1.
      const int LM = 1 << lb;
      o << "      const bool h = (lane >> " << lb << ") & 1; const " << (prec == 0 ? "float" : "double")
        << " sg = h ? -1 : 1;\n";
      bool need[8][2] = {};
      for (int p = 0; p < P; ++p) need[unit_of(p)][st_parity(am, p)] = true;
      for (int u = 0; u < UNR; ++u)
        for (int s = 0; s < 2; ++s) {
          if (!need[u][s]) continue;
          if (prec == 0)
            o << "      const float c" << u << s << " = h ? " << (s ? "-" : "") << "ar" << u << " : " << (fold ? "sck" : "1.f")
              << "; const u64 cB" << u << s << " = h ? (B" << u << (s ? " ^ OWQS_SIGN2" : "") << ") : 0ull;\n";
          else
            o << "      const double cr" << u << s << " = h ? " << (s ? "-" : "") << "ar" << u << " : " << (fold ? "sck" : "1.0")
              << ", ci" << u << s << " = h ? " << (s ? "-" : "") << "ai" << u << " : 0.0;\n";
        }
      for (int p = 0; p < P; ++p) {
        const int u = unit_of(p), s = st_parity(am, p);
        if (prec == 0) {
          o << "      { const u64 y = fma2(cB" << u << s << ", swp(" << X(p) << "), mul2(bc(c" << u << s << "), " << X(p)
            << ")); " << X(p) << " = fma2(bc(sg), y, shfl2(y, " << LM << ")); }\n";
        } else {
          const std::string c = std::to_string(u) + std::to_string(s);
          o << "      { const double yr = cr" << c << " * " << XR(p) << " - ci" << c << " * " << XI(p) << ", yi = cr" << c
            << " * " << XI(p) << " + ci" << c << " * " << XR(p) << "; " << XR(p) << " = __shfl_xor_sync(0xffffffffu, yr, "
            << LM << ") + sg * yr; " << XI(p) << " = __shfl_xor_sync(0xffffffffu, yi, " << LM << ") + sg * yi; }\n";
        }
      }
    } else {
      error = "butterfly on a slot outside the thread's registers and lanes";
    }
    o << "    }\n";
  }

  void xop(int i) {
    const Op& op = d.ops[i];
    const int a = op.a;
    int lb;
    const int ka = kind(a, &lb);
    o << "    // op " << i << ": X on slot " << a << (op.cond ? " (conditional)" : "") << "\n";
    if (ka == SK_REG) {
      const int pb = lb;
      if (!op.cond) {  // compile-time renaming
        for (int p = 0; p < P; ++p)
          if (!(p & pb)) std::swap(perm[p], perm[p | pb]);
        return;
      }
      o << "    if (" << cond_expr(i) << ") {\n";
      for (int p = 0; p < P; ++p) {
        if (p & pb) continue;
        const int p1 = p | pb;
        if (prec == 0)
          o << "      { const u64 t = " << X(p) << "; " << X(p) << " = " << X(p1) << "; " << X(p1) << " = t; }\n";
        else
          o << "      { const double tr = " << XR(p) << ", ti = " << XI(p) << "; " << XR(p) << " = " << XR(p1) << "; "
            << XI(p) << " = " << XI(p1) << "; " << XR(p1) << " = tr; " << XI(p1) << " = ti; }\n";
      }
      o << "    }\n";
    } else if (ka == SK_LANE) {
      const std::string lm =
          op.cond ? "(" + cond_expr(i) + " ? " + std::to_string(1 << lb) + " : 0)" : std::to_string(1 << lb);
      o << "    { const int lm = " << lm << ";\n";
      for (int p = 0; p < P; ++p) {
        if (prec == 0)
          o << "      " << X(p) << " = shfl2(" << X(p) << ", lm);\n";
        else
          o << "      " << XR(p) << " = __shfl_xor_sync(0xffffffffu, " << XR(p) << ", lm); " << XI(p)
            << " = __shfl_xor_sync(0xffffffffu, " << XI(p) << ", lm);\n";
      }
      o << "    }\n";
    } else {
      error = "X on a slot outside the thread's registers and lanes";
    }
  }

  // apply the pending diagonal sign flips (E = CZ, Z^s): sign of an amplitude = XOR over pending
  // ops whose register bits are all 1 there of (cond AND the op's runtime bits)
  void flush() {
    if (pend.empty()) return;
    o << "    {  // flush " << pend.size() << " pending diagonal(s)\n";
    struct Term {
      std::vector<int> regs;
      bool stat1;
      std::vector<std::string> rt;
    };
    std::vector<Term> terms;
    for (size_t k = 0; k < pend.size(); ++k) {
      const Pend& pe = pend[k];
      Term t;
      std::vector<int> slots = {pe.a};
      if (pe.b != pe.a) slots.push_back(pe.b);
      std::vector<int> rts;
      for (int s : slots) (is_reg(s) ? t.regs : rts).push_back(s);
      t.stat1 = rts.empty() && !pe.cond;
      if (!t.stat1)
        for (int u = 0; u < UNR; ++u) {
          std::string nm = "f" + std::to_string(k) + "_" + std::to_string(u);
          std::string e = pe.cond ? "(unsigned)" + cond_expr(pe.idx) : "1u";
          for (int s : rts) e += " & " + rt_bit(s, u);
          o << "      const unsigned " << nm << " = " << e << ";\n";
          t.rt.push_back(nm);
        }
      terms.push_back(t);
    }
    for (int p = 0; p < P; ++p) {
      int stat = 0;
      std::vector<std::string> dyn;
      for (const Term& t : terms) {
        bool on = true;
        for (int s : t.regs) on = on && regval(s, p);
        if (!on) continue;
        if (t.stat1)
          stat ^= 1;
        else
          dyn.push_back(t.rt[unit_of(p)]);
      }
      if (dyn.empty() && !stat) continue;
      if (dyn.empty()) {
        if (prec == 0)
          o << "      " << X(p) << " ^= OWQS_SIGN2;\n";
        else
          o << "      " << XR(p) << " = -" << XR(p) << "; " << XI(p) << " = -" << XI(p) << ";\n";
        continue;
      }
      std::string f = stat ? "1u" : "0u";
      for (auto& s : dyn) f += " ^ " + s;
      if (prec == 0)
        o << "      " << X(p) << " = flip2(" << X(p) << ", " << f << ");\n";
      else
        o << "      { const unsigned f = " << f << "; " << XR(p) << " = fld(" << XR(p) << ", f); " << XI(p) << " = fld("
          << XI(p) << ", f); }\n";
    }
    o << "    }\n";
    pend.clear();
  }

  void reduce() {
    if (d.red_kind == RED_NONE) return;
    if (d.red_kind == RED_NORM) {
      if (prec == 0) {
        o << "    { u64 n0 = 0ull, n1 = 0ull;\n";
        for (int p = 0; p < P; ++p) o << "      n" << (p & 1) << " = fma2(" << X(p) << ", " << X(p) << ", n" << (p & 1) << ");\n";
        o << "      const u64 n = add2(n0, n1); acc0 += (double)lo(n) + (double)hi(n); }\n";
      } else {
        o << "    { double n0 = 0.0, n1 = 0.0;\n";
        for (int p = 0; p < P; ++p)
          o << "      n" << (p & 1) << " += " << XR(p) << " * " << XR(p) << " + " << XI(p) << " * " << XI(p) << ";\n";
        o << "      acc0 += n0 + n1; }\n";
      }
      return;
    }
    // RED_RHO on slot r: n0 = sum |x|^2 over bit r = 0, n1 over bit r = 1, c = sum conj(x0) x1
    const int r = d.red_slot;
    int lb;
    const int kr = kind(r, &lb);
    if (kr == SK_REG) {
      const int pb = lb;
      if (prec == 0) {
        o << "    { u64 n0 = 0ull, n1 = 0ull, cc = 0ull, cd = 0ull;\n";
        for (int p = 0; p < P; ++p) {
          if (p & pb) continue;
          const int p1 = p | pb;
          o << "      n0 = fma2(" << X(p) << ", " << X(p) << ", n0); n1 = fma2(" << X(p1) << ", " << X(p1)
            << ", n1); cc = fma2(" << X(p) << ", " << X(p1) << ", cc); cd = fma2(" << X(p) << ", swp(" << X(p1)
            << "), cd);\n";
        }
        o << "      acc0 += (double)lo(n0) + (double)hi(n0); acc1 += (double)lo(n1) + (double)hi(n1);\n"
             "      acc2 += (double)lo(cc) + (double)hi(cc); acc3 += (double)lo(cd) - (double)hi(cd); }\n";
      } else {
        o << "    {\n";
        for (int p = 0; p < P; ++p) {
          if (p & pb) continue;
          const int p1 = p | pb;
          o << "      acc0 += " << XR(p) << " * " << XR(p) << " + " << XI(p) << " * " << XI(p) << "; acc1 += " << XR(p1)
            << " * " << XR(p1) << " + " << XI(p1) << " * " << XI(p1) << "; acc2 += " << XR(p) << " * " << XR(p1)
            << " + " << XI(p) << " * " << XI(p1) << "; acc3 += " << XR(p) << " * " << XI(p1) << " - " << XI(p)
            << " * " << XR(p1) << ";\n";
        }
        o << "    }\n";
      }
    } else if (kr == SK_LANE) {
      const int LM = 1 << lb;
      if (prec == 0) {
        o << "    { u64 nn = 0ull, cc = 0ull, cd = 0ull;\n";
        for (int p = 0; p < P; ++p)
          o << "      { const u64 q = shfl2(" << X(p) << ", " << LM << "); nn = fma2(" << X(p) << ", " << X(p)
            << ", nn); cc = fma2(" << X(p) << ", q, cc); cd = fma2(" << X(p) << ", swp(q), cd); }\n";
        o << "      const double nd = (double)lo(nn) + (double)hi(nn);\n"
             "      if ((lane >> " << lb << ") & 1) { acc1 += nd; } else { acc0 += nd; acc2 += (double)lo(cc) + (double)hi(cc); acc3 += (double)lo(cd) - (double)hi(cd); } }\n";
      } else {
        o << "    { double nn = 0.0, cc = 0.0, cd = 0.0;\n";
        for (int p = 0; p < P; ++p)
          o << "      { const double qr = __shfl_xor_sync(0xffffffffu, " << XR(p) << ", " << LM
            << "), qi = __shfl_xor_sync(0xffffffffu, " << XI(p) << ", " << LM << "); nn += " << XR(p) << " * " << XR(p)
            << " + " << XI(p) << " * " << XI(p) << "; cc += " << XR(p) << " * qr + " << XI(p) << " * qi; cd += " << XR(p)
            << " * qi - " << XI(p) << " * qr; }\n";
        o << "      if ((lane >> " << lb << ") & 1) { acc1 += nn; } else { acc0 += nn; acc2 += cc; acc3 += cd; } }\n";
      }
    } else {
      error = "reduction slot outside the thread's registers and lanes";
    }
  }

  // unit index -> group base (zeros inserted at the group slots, ascending)
  void emit_gb(const std::string& dst, const std::string& unit) {
    o << "    unsigned long long " << dst << " = " << unit << ";\n";
    for (int j = 0; j < KHI; ++j) {
      const int q = gs[j] - SB;
      o << "    " << dst << " = ((" << dst << " >> " << q << ") << " << (q + 1) << ") | (" << dst << " & "
        << ((1ull << q) - 1) << "ull);\n";
    }
  }
  uint64_t seg_off(int c) const {
    uint64_t s = 0;
    for (int j = 0; j < KHI; ++j)
      if ((c >> j) & 1) s |= 1ull << (gs[j] - SB);
    return s;
  }

  void emit_op(int i, int bi) {
    const Op& op = d.ops[i];
    switch (op.type) {
      case OP_DIAG_E:
      case OP_DIAG_Z:
        pend.push_back({op.a, op.type == OP_DIAG_E ? op.b : op.a, i, op.cond != 0});
        break;
      case OP_FLUSH:
        flush();
        break;
      case OP_X:
        xop(i);
        break;
      case OP_BFLY:
        bfly(i, bi);
        break;
      default:
        break;
    }
  }

  // ---- engine 1: direct coalesced loads into registers (complex128, and narrow complex64) ----
  std::string run_direct() {
    const int nbf = d.n_bfly;
    const int red = d.red_kind;
    const int nred = red == RED_NONE ? 0 : (red == RED_NORM ? 1 : 4);
    const int minb = KHI <= 3 ? 3 : 2;
    const int slack = d.width - SB - KHI - (UNR == 4 ? 2 : (UNR == 2 ? 1 : 0)) - 3;
    const uint64_t nbu = 1ull << slack;
    o << "extern \"C\" __global__ void __launch_bounds__(256, " << minb << ") OWQS_KNAME(const owqs::StepDesc d, const owqs::DevPtrs p) {\n"
      << "  using namespace owqs;\n"
      << "  // direct engine: width " << d.width << ", group slots";
    for (int j = 0; j < KHI; ++j) o << " " << gs[j];
    o << ", " << d.n_ops << " ops, " << nbf << " butterflies, reduction " << red << "\n";
    o << "  __shared__ PassShared sh;\n";
    if (prec == 0)
      o << "  __shared__ float s_ar[" << std::max(1, nbf) << "]; __shared__ u64 s_B[" << std::max(1, nbf) << "];\n";
    else
      o << "  __shared__ double s_ar[" << std::max(1, nbf) << "], s_ai[" << std::max(1, nbf) << "];\n";
    o << "  pass_prologue(d, p, sh);\n";
    if (nbf > 0) {
      o << "  for (int b = threadIdx.x; b < " << nbf << "; b += blockDim.x) {\n";
      if (prec == 0)
        o << "    const float ai = (float)sh.ka[b][1]; s_ar[b] = (float)sh.ka[b][0]; s_B[b] = pk(-ai, ai);\n";
      else
        o << "    s_ar[b] = sh.ka[b][0]; s_ai[b] = sh.ka[b][1];\n";
      o << "  }\n  __syncthreads();\n";
    }
    o << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
      << "  const unsigned rk = p.rank; (void)rk;\n"
      << "  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;\n";
    if (nbf > 0) {
      if (prec == 0)
        o << "  const u64 scale = bc((float)sh.scale);\n";
      else
        o << "  const double scale = sh.scale;\n";
    }
    if (prec == 0)
      o << "  float4* __restrict__ st = reinterpret_cast<float4*>(p.state);\n";
    else
      o << "  double2* __restrict__ st = reinterpret_cast<double2*>(p.state);\n";
    o << "  for (unsigned long long ub = blockIdx.x; ub < " << nbu << "ull; ub += gridDim.x) {\n"
      << "    const unsigned long long unit = ub * 8 + warp;\n";
    for (int u = 0; u < UNR; ++u) emit_gb("gb" + std::to_string(u), "unit * " + std::to_string(UNR) + " + " + std::to_string(u));
    for (int u = 0; u < UNR; ++u)
      for (int c = 0; c < G; ++c) {
        const int v = u * G + c;
        const std::string addr = "st + (((gb" + std::to_string(u) + " | " + std::to_string(seg_off(c)) + "ull) << 5) + lane)";
        if (prec == 0)
          o << "    u64 x" << 2 * v << ", x" << 2 * v + 1 << "; { const float4 w = __ldcs(" << addr << "); x" << 2 * v
            << " = pk(w.x, w.y); x" << 2 * v + 1 << " = pk(w.z, w.w); }\n";
        else
          o << "    double xr" << v << ", xi" << v << "; { const double2 w = __ldcs(" << addr << "); xr" << v
            << " = w.x; xi" << v << " = w.y; }\n";
      }
    int bi = 0;
    for (int i = 0; i < d.n_ops; ++i) emit_op(i, d.ops[i].type == OP_BFLY ? bi++ : -1);
    flush();
    emit_scale(nbf);
    reduce();
    if (d.n_ops > 0) {
      for (int u = 0; u < UNR; ++u)
        for (int c = 0; c < G; ++c) {
          const int v = u * G + c;
          const std::string addr = "st + (((gb" + std::to_string(u) + " | " + std::to_string(seg_off(c)) + "ull) << 5) + lane)";
          const int p0 = v * EPV;
          if (prec == 0)
            o << "    __stcs(" << addr << ", make_float4(lo(" << X(p0) << "), hi(" << X(p0) << "), lo(" << X(p0 + 1)
              << "), hi(" << X(p0 + 1) << ")));\n";
          else
            o << "    __stcs(" << addr << ", make_double2(" << XR(p0) << ", " << XI(p0) << "));\n";
        }
    }
    o << "  }\n";
    if (nred > 0) o << "  double acc[4] = {acc0, acc1, acc2, acc3};\n  reduce_finish<" << nred << ">(acc, p, sh);\n";
    o << "}\n";
    return o.str();
  }

  bool scale_pending = false;
  void emit_scale(int nbf) {
    if (nbf == 0 || (tile && !scale_pending)) return;
    for (int p = 0; p < P; ++p) {
      if (prec == 0)
        o << "    " << X(p) << " = mul2(scale, " << X(p) << ");\n";
      else
        o << "    " << XR(p) << " *= scale; " << XI(p) << " *= scale;\n";
    }
  }

  // ---- engine 2: phase planning ---------------------------------------------------------------
  // ops of the pass in a dependency DAG (two ops conflict when one's non-diagonal slot is touched
  // by the other; diagonals commute; FLUSH is a barrier); index n = the reduction (after all).
  // A phase = a register set (t0 + 4 tile bits) and the ops it runs; greedy: each phase picks the
  // 4 tile bits that let the most ready ops run, one bit at a time.
  struct Phase {
    int S[5];  // S[0..RB-2]: register tile bits besides t0
    std::vector<int> ops;
  };
  int n_ops_ = 0;
  std::vector<std::vector<int>> preds;
  std::vector<int> op_tb;  // tile bit an op needs in registers (-1: none)
  uint64_t tile_iters = 1;
  // CTAs per SM the tile kernel is compiled for (register cap 65536 / (256 * minb)). 2: measured on
  // C3, 3 (80 registers) is 18% slower (serialised loads)
  static int tile_minb_for(int prec) {
    const char* e = getenv("OWQS_TILE_MINB");
    if (e) return std::max(1, std::min(8, atoi(e)));
    if (tile_g(prec) < KTILE) return 2 << (KTILE - tile_g(prec));  // 4- / 2-warp CTAs
    return (prec == 0 && tile_geom().rb == 6) ? 3 : 2;
  }
  int tile_minb() const { return tile_minb_for(prec); }
  int n_local_ = 0, n_cta_ = 0, n_group_ = 0, next_bar_ = 1;

  void build_dag() {
    const int n = d.n_ops;
    n_ops_ = n;
    preds.assign(n + 1, {});
    op_tb.assign(n + 1, -1);
    std::vector<uint64_t> nd(n + 1, 0), dg(n + 1, 0);
    std::vector<char> bar(n + 1, 0);
    int bi = 0;
    for (int i = 0; i < n; ++i) {
      const Op& op = d.ops[i];
      if (op.type == OP_BFLY) {
        nd[i] = 1ull << op.a;
        dg[i] = d.absorb[bi++];
        op_tb[i] = tilebit(op.a);
      } else if (op.type == OP_X) {
        nd[i] = 1ull << op.a;
        op_tb[i] = tilebit(op.a);
      } else if (op.type == OP_DIAG_E) {
        dg[i] = (1ull << op.a) | (1ull << op.b);
      } else if (op.type == OP_DIAG_Z) {
        dg[i] = 1ull << op.a;
      } else if (op.type == OP_FLUSH) {
        bar[i] = 1;
      }
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j)
        if (bar[i] || bar[j] || (nd[j] & (nd[i] | dg[i])) || (dg[j] & nd[i])) preds[i].push_back(j);
    for (int j = 0; j < n; ++j) preds[n].push_back(j);
    if (d.red_kind == RED_RHO) op_tb[n] = tilebit(d.red_slot);
  }
  bool exec_in(int i, unsigned regmask) const { return op_tb[i] < 0 || ((regmask >> op_tb[i]) & 1); }
  // ops (ascending) that run in a phase with register tile-bit mask regmask, given done
  std::vector<int> closure(unsigned regmask, const std::vector<char>& done) const {
    std::vector<char> take(n_ops_ + 1, 0);
    std::vector<int> out;
    for (int i = 0; i <= n_ops_; ++i) {
      if (done[i] || !exec_in(i, regmask)) continue;
      bool ok = true;
      for (int j : preds[i])
        if (!done[j] && !take[j]) {
          ok = false;
          break;
        }
      if (ok) {
        take[i] = 1;
        out.push_back(i);
      }
    }
    return out;
  }
  // Phases: each picks, among all C(12, 4) register sets (t0 + 4 of t1..t12), the one that runs the
  // most ready ops (ties: fewer bits outside the pass's preferred warp bits, then A-type sets).
  // Bitset form of the DAG for the phase search (ops + the reduction <= 128).
  struct Bits {
    uint64_t w[3] = {0, 0, 0};
    void set(int i) { w[i >> 6] |= 1ull << (i & 63); }
    bool get(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
    bool disjoint(const Bits& o) const { return !(w[0] & o.w[0]) && !(w[1] & o.w[1]) && !(w[2] & o.w[2]); }
    int count() const { return __builtin_popcountll(w[0]) + __builtin_popcountll(w[1]) + __builtin_popcountll(w[2]); }
  };
  std::vector<Bits> predbits;
  void build_predbits() {
    predbits.assign(n_ops_ + 1, Bits());
    for (int i = 0; i <= n_ops_; ++i)
      for (int j : preds[i]) predbits[i].set(j);
  }
  // ops runnable in a phase with register mask regs after `done`: closure in op order
  Bits closure_bits(unsigned regs, const Bits& done) const {
    Bits take = done;
    for (int i = 0; i <= n_ops_; ++i) {
      if (done.get(i) || !exec_in(i, regs)) continue;
      const Bits& pb = predbits[i];
      // every predecessor done or taken: pb & ~take == 0
      if ((pb.w[0] & ~take.w[0]) || (pb.w[1] & ~take.w[1]) || (pb.w[2] & ~take.w[2])) continue;
      take.set(i);
    }
    return take;
  }
  // Beam search over phase sequences: each step expands a state by the register sets that run the
  // most ready ops (top kExpand), keeps the kBeam states with the most ops done, and stops at the
  // first depth where a state has run every op; ties go to fewer transposes (non-A first/last
  // phases cost one each). first_group_only: the first phase must be loadable (A-type).
  std::vector<Phase> plan_greedy(bool first_group_only) const {
    static const int kBeam = getenv("OWQS_BEAM") ? atoi(getenv("OWQS_BEAM")) : 8;
    static const int kExpand = getenv("OWQS_EXPAND") ? atoi(getenv("OWQS_EXPAND")) : 6;
    struct St {
      Bits done;
      std::vector<Phase> ph;
    };
    std::vector<unsigned> sets;
    std::vector<std::array<int, 5>> setS;
    for (unsigned m = 0; m < (1u << (TB - FB)); ++m) {
      if (__builtin_popcount(m) != NSEL) continue;
      const unsigned regs = (FB ? 1u : 0u) | (m << FB);
      static const bool wregs = getenv("OWQS_WARP_IN_REGS") != nullptr;
      if (!wregs && (regs & warp_pref)) continue;  // keep the pass's warp bits out of registers
      std::array<int, 5> S{};
      int n = 0;
      for (int b = FB; b < TB; ++b)
        if ((regs >> b) & 1) S[n++] = b;
      sets.push_back(regs);
      setS.push_back(S);
    }
    std::vector<St> beam(1);
    const int total = n_ops_ + 1;
    for (int depth = 0; depth < 64; ++depth) {
      std::vector<St> next;
      for (const St& st : beam) {
        const int have = st.done.count();
        std::vector<std::pair<int, int>> cand;  // (gain * 2 + a_type, set index)
        for (size_t k = 0; k < sets.size(); ++k) {
          if (depth == 0 && first_group_only && !a_type(setS[k].data())) continue;
          const int gain = closure_bits(sets[k], st.done).count() - have;
          if (gain > 0) cand.push_back({gain * 2 + (a_type(setS[k].data()) ? 1 : 0), (int)k});
        }
        std::sort(cand.begin(), cand.end(), [](auto& x, auto& y) { return x.first > y.first; });
        for (int c = 0; c < (int)cand.size() && c < kExpand; ++c) {
          St ns = st;
          const int k = cand[c].second;
          Phase f{};
          for (int j = 0; j < NSEL; ++j) f.S[j] = setS[k][j];
          const Bits nd = closure_bits(sets[k], st.done);
          for (int i = 0; i <= n_ops_; ++i)
            if (nd.get(i) && !st.done.get(i)) f.ops.push_back(i);
          ns.done = nd;
          ns.ph.push_back(f);
          next.push_back(ns);
        }
      }
      if (next.empty()) return {};
      std::vector<const St*> fin;
      for (const St& st : next)
        if (st.done.count() == total) fin.push_back(&st);
      if (!fin.empty()) {
        const St* best = fin[0];
        for (const St* f : fin)
          if (n_transitions(f->ph) < n_transitions(best->ph)) best = f;
        return best->ph;
      }
      std::stable_sort(next.begin(), next.end(), [](const St& x, const St& y) { return x.done.count() > y.done.count(); });
      // drop duplicates (same done set)
      std::vector<St> keep;
      for (const St& st : next) {
        bool dup = false;
        for (const St& k2 : keep)
          if (!memcmp(k2.done.w, st.done.w, sizeof st.done.w) && k2.ph.back().S[0] == st.ph.back().S[0] &&
              !memcmp(k2.ph.back().S, st.ph.back().S, sizeof st.ph.back().S)) {
            dup = true;
            break;
          }
        if (!dup) keep.push_back(st);
        if ((int)keep.size() >= kBeam) break;
      }
      beam.swap(keep);
    }
    return {};
  }
  // the pass's warp bits: the 3 group tile bits with the fewest non-diagonal ops (untouched padding
  // slots first), so that phase changes keep them and transpose within each warp
  unsigned warp_pref = 0;
  void choose_warp_bits() {
    std::vector<int> use(TB, 0);
    for (int i = 0; i <= n_ops_; ++i)
      if (op_tb[i] >= 0) ++use[op_tb[i]];
    std::vector<int> cand;
    for (int b = SB; b < TB; ++b) cand.push_back(b);
    std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) { return use[x] < use[y]; });
    warp_pref = 0;
    for (int k = 0; k < WB; ++k) warp_pref |= 1u << cand[k];
    // a bit needed in registers by some op cannot be a warp bit for the whole pass: drop it
    for (int k = 0; k < WB; ++k)
      if (use[cand[k]] > 0) warp_pref &= ~(1u << cand[k]);
  }
  bool a_type(const int* S) const {
    if (t0free) {  // t0 + 4 group bits (global IO pairs t0 neighbours in float4)
      bool has0 = false;
      for (int k = 0; k < NSEL; ++k) {
        if (S[k] == 0) has0 = true;
        else if (S[k] < SB) return false;
      }
      return has0;
    }
    for (int k = 0; k < NSEL; ++k)
      if (S[k] < SB) return false;
    return true;
  }
  int n_transitions(const std::vector<Phase>& ph) const {
    if (ph.empty()) return 1 << 20;
    int t = (int)ph.size() - 1;
    if (!a_type(ph.front().S)) ++t;
    if (!a_type(ph.back().S)) ++t;
    return t;
  }
  // lanes / warps for a register set
  CLayout make_layout(const int* S) const {
    CLayout L;
    for (int k = 0; k < FB; ++k) L.R[k] = k;  // complex64: t0 in R[0]
    for (int k = 0; k < NSEL; ++k) L.R[FB + k] = S[k];
    auto in_s = [&](int b) {
      for (int k = 0; k < RB; ++k)
        if (L.R[k] == b) return true;
      return false;
    };
    // warp bits: the pass's preferred ones first (ascending), then the highest free group bits
    int w = 0;
    for (int b = SB; b < TB && w < WB; ++b)
      if (((warp_pref >> b) & 1) && !in_s(b)) L.Wb[w++] = b;
    for (int b = TB - 1; b >= SB && w < WB; --b) {
      bool taken = in_s(b);
      for (int j = 0; j < w; ++j) taken = taken || L.Wb[j] == b;
      if (!taken) L.Wb[w++] = b;
    }
    if (w < WB)  // S holds group bits and the preferred set overlaps: any remaining bits
      for (int b = TB - 1; b >= (prec == 0 ? 1 : 0) && w < WB; --b) {
        bool taken = in_s(b);
        for (int j = 0; j < w; ++j) taken = taken || L.Wb[j] == b;
        if (!taken) L.Wb[w++] = b;
      }
    std::sort(L.Wb, L.Wb + WB);
    auto in_w = [&](int b) {
      for (int j = 0; j < WB; ++j)
        if (L.Wb[j] == b) return true;
      return false;
    };
    bool seg_lanes = a_type(S);
    for (int j = 0; j < 5; ++j) seg_lanes = seg_lanes && !in_w(LS + j);
    if (seg_lanes) {  // A-type: lanes = the segment's lane slots (global IO layout)
      for (int j = 0; j < 5; ++j) L.Lb[j] = LS + j;
      return L;
    }
    std::vector<int> rest;
    for (int b = (t0free ? 1 : 0); b < TB; ++b)  // t0 (when not a register bit) goes to lane bit 3
      if (!in_s(b) && !in_w(b)) rest.push_back(b);
    // lane bits 0..2: one tile bit of each bank class, lowest first
    std::vector<char> used(rest.size(), 0);
    for (int c = 0; c < 3; ++c) {
      int pick = -1;
      for (size_t i = 0; i < rest.size(); ++i)
        if (!used[i] && bclass(rest[i]) == c) {
          pick = (int)i;
          break;
        }
      if (pick < 0)  // no bit of this class left: 2-way bank conflicts, still correct
        for (size_t i = 0; i < rest.size(); ++i)
          if (!used[i]) {
            pick = (int)i;
            break;
          }
      used[pick] = 1;
      L.Lb[c] = rest[pick];
    }
    int j = 3;
    if (t0free && !in_s(0)) L.Lb[j++] = 0;
    for (size_t i = 0; i < rest.size(); ++i)
      if (!used[i] && j < 5) L.Lb[j++] = rest[i];
    return L;
  }
  int treg(const CLayout& L, int p) const {
    int t = 0;
    for (int k = 0; k < RB; ++k)
      if ((p >> k) & 1) t |= 1 << L.R[k];
    return t;
  }
  int add_layout(const CLayout& L) {
    for (size_t i = 0; i < lays.size(); ++i)
      if (!memcmp(&lays[i], &L, sizeof L)) return (int)i;
    lays.push_back(L);
    return (int)lays.size() - 1;
  }
  // global slot of each tile bit: the pass's slots, or (store side) after the pass's qubit remap
  int slot_of_tb(int t) const { return t < SB ? t : gs[t - SB]; }
  int smap[16];
  bool use_smap = false;
  int gslot(int t) const { return use_smap ? smap[t] : slot_of_tb(t); }
  // segment offset (relative to gb) of register pair p in A-type layout l (group bits only)
  uint64_t a_seg(int l, int p) const {
    uint64_t s = 0;
    const CLayout& L = lays[l];
    for (int k = 0; k < RB; ++k)
      if (((p >> k) & 1) && gslot(L.R[k]) >= SB) s |= 1ull << (gslot(L.R[k]) - SB);
    return s;
  }
  // global float4/double2 offset of a lane in the store layout: lane bit i -> segment slot smap[Lb[i]]
  std::string lane_expr(const CLayout& L, bool remapped) const {
    std::string e = "(0";
    bool ident = true;
    for (int i = 0; i < 5; ++i) {
      const int j = (remapped ? smap[L.Lb[i]] : slot_of_tb(L.Lb[i])) - LS;
      ident = ident && j == i;
      e += " | (((lane >> " + std::to_string(i) + ") & 1) << " + std::to_string(j) + ")";
    }
    return ident ? "lane" : e + ")";
  }
  // store layout under the remap: lanes = the tile bits that land on the segment's lane slots,
  // registers = t0 (complex64) + the last phase's other bits where possible, warps = the rest
  CLayout make_store_layout(const CLayout& last) const {
    CLayout L;
    bool used[16] = {};
    // lanes = the tile bits stored to the segment's 5 lane slots, ordered so that lane bits 0..2
    // carry one bank class each where possible (a quarter-warp's 16 B accesses conflict-free); any
    // order covers the same 512 B, the store offset follows the permutation (store_lane_expr)
    int seg[5];
    for (int j = 0; j < 5; ++j)
      for (int t = 0; t < TB; ++t)
        if (smap[t] == LS + j) seg[j] = t;
    bool taken[5] = {};
    int li = 0;
    for (int c = 0; c < 3; ++c)
      for (int j = 0; j < 5; ++j)
        if (!taken[j] && bclass(seg[j]) == c) {
          taken[j] = true;
          L.Lb[li++] = seg[j];
          break;
        }
    for (int j = 0; j < 5; ++j)
      if (!taken[j]) L.Lb[li++] = seg[j];
    for (int j = 0; j < 5; ++j) used[L.Lb[j]] = true;
    int k = 0;
    const int fb = prec == 0 ? 1 : 0;  // global stores pair t0 neighbours (float4)
    if (fb) {
      L.R[k++] = 0;
      used[0] = true;
    }
    for (int q = 0; q < RB && k < RB; ++q)
      if (!used[last.R[q]]) {
        L.R[k++] = last.R[q];
        used[last.R[q]] = true;
      }
    for (int t = 0; t < TB && k < RB; ++t)
      if (!used[t]) {
        L.R[k++] = t;
        used[t] = true;
      }
    int w = 0;
    for (int t = 0; t < TB; ++t)
      if (!used[t]) L.Wb[w++] = t;
    std::sort(L.R + fb, L.R + RB);
    return L;
  }
  void emit_tile_transition(int to, bool last) {
    o << "    // layout " << lay << " -> " << to << " (shared-memory tile)\n";
    const CLayout& A = lays[lay];
    const CLayout& B = lays[to];
    // warp bits unchanged: every warp exchanges only its own amplitudes (warp-local barrier)
    const bool local = !memcmp(A.Wb, B.Wb, sizeof(int) * WB);
    // otherwise only the warps that exchange amplitudes synchronise: the connected components of
    // {writer warp of t (layout A), reader warp of t (layout B)} over the tile's indices t -- cosets of
    // the warp-index bits both layouts assign to the same tile bit -- each on its own named barrier
    std::string bar = local ? "    __syncwarp();\n" : "    __syncthreads();\n";
    if (!local && !getenv("OWQS_NO_GROUPBAR")) {
      const int NW = 1 << WB;
      int comp[8];
      for (int w = 0; w < NW; ++w) comp[w] = w;
      std::function<int(int)> find = [&](int x) { return comp[x] == x ? x : comp[x] = find(comp[x]); };
      for (int t = 0; t < (1 << TB); ++t) {
        int wa = 0, wb = 0;
        for (int j = 0; j < WB; ++j) {
          wa |= ((t >> A.Wb[j]) & 1) << j;
          wb |= ((t >> B.Wb[j]) & 1) << j;
        }
        const int ra = find(wa), rb = find(wb);
        if (ra != rb) comp[std::max(ra, rb)] = std::min(ra, rb);
      }
      int size[8] = {}, id[8], nid = 0, rep_id[8];
      for (int w = 0; w < NW; ++w) ++size[find(w)];
      for (int w = 0; w < NW; ++w)
        if (find(w) == w) rep_id[w] = nid++;
      bool uniform = true;
      for (int w = 0; w < NW; ++w) {
        id[w] = rep_id[find(w)];
        uniform = uniform && size[find(w)] == size[find(0)];
      }
      if (uniform && nid > 1) {
        // fresh barrier ids for every grouped transpose: a warp may run ahead into the next
        // transpose while others still wait on this one's barrier, so an id is reused only after a
        // CTA-wide barrier (bar 0) has been passed by all warps
        std::string pre;
        if (next_bar_ + nid > 16) {
          pre = "    __syncthreads();\n";
          next_bar_ = 1;
        }
        uint32_t table = 0;
        for (int w = 0; w < NW; ++w) table |= (uint32_t)(next_bar_ + id[w]) << (4 * w);
        next_bar_ += nid;
        bar = pre + "    asm volatile(\"bar.sync %0, %1;\" :: \"r\"((" + std::to_string(table) +
              "u >> (4 * warp)) & 15), \"r\"(" + std::to_string(32 * size[find(0)]) + ") : \"memory\");\n";
        ++n_group_;
      }
    }
    if (bar == "    __syncthreads();\n") next_bar_ = 1;
    if (prec == 0) {
      // t0 in register position 0: 16 B accesses of t0 neighbours; else 8 B per amplitude
      if (A.R[0] == 0)
        for (int p = 0; p < P; p += 2)
          o << "    *reinterpret_cast<float4*>(dsm + (sb" << lay << " ^ " << addrb(treg(A, p)) << ")) = make_float4(lo("
            << X(p) << "), hi(" << X(p) << "), lo(" << X(p + 1) << "), hi(" << X(p + 1) << "));\n";
      else
        for (int p = 0; p < P; ++p)
          o << "    *reinterpret_cast<float2*>(dsm + (sb" << lay << " ^ " << addrb(treg(A, p)) << ")) = make_float2(lo("
            << X(p) << "), hi(" << X(p) << "));\n";
      o << bar;
      if (B.R[0] == 0)
        for (int p = 0; p < P; p += 2)
          o << "    { const float4 w = *reinterpret_cast<const float4*>(dsm + (sb" << to << " ^ " << addrb(treg(B, p))
            << ")); x" << p << " = pk(w.x, w.y); x" << p + 1 << " = pk(w.z, w.w); }\n";
      else
        for (int p = 0; p < P; ++p)
          o << "    { const float2 w = *reinterpret_cast<const float2*>(dsm + (sb" << to << " ^ " << addrb(treg(B, p))
            << ")); x" << p << " = pk(w.x, w.y); }\n";
    } else {
      for (int p = 0; p < P; ++p)
        o << "    *reinterpret_cast<double2*>(dsm + (sb" << lay << " ^ " << addrb(treg(A, p)) << ")) = make_double2("
          << XR(p) << ", " << XI(p) << ");\n";
      o << bar;
      for (int p = 0; p < P; ++p)
        o << "    { const double2 w = *reinterpret_cast<const double2*>(dsm + (sb" << to << " ^ " << addrb(treg(B, p))
          << ")); xr" << p << " = w.x; xi" << p << " = w.y; }\n";
    }
    for (int p = 0; p < P; ++p) perm[p] = p;
    // no write-after-read barrier between transposes: location u(t) depends only on the tile index
    // t, and the thread that writes it in the next transpose is the one that read it in this one.
    // Only a next tile of the same CTA (other writers) needs one.
    if ((last && tile_iters > 1) || (!last && getenv("OWQS_TRANS_WAR"))) o << "    __syncthreads();\n";
    ++(local ? n_local_ : n_cta_);
    lay = to;
  }

  // ---- engine 2 kernel: one CTA = one 13-bit tile (non-persistent grid), coalesced global IO in
  // A-type layouts, phases separated by shared-memory transposes, decisions from PassCoef,
  // deterministic two-level grid reduction ----
  std::string run_tile() {
    const int nbf = d.n_bfly;
    const bool small = jit_tile_small(d, prec);
    const int red = d.red_kind;
    const int nred = red == RED_NONE ? 0 : (red == RED_NORM ? 1 : 4);
    const uint64_t nbu = 1ull << (d.width - TB);
    const uint64_t iters = nbu / jit_tile_blocks(d, prec);
    tile_iters = iters;
    build_dag();
    build_predbits();
    choose_warp_bits();
    std::vector<Phase> pa = plan_greedy(true), pb = plan_greedy(false);
    const std::vector<Phase>& ph = n_transitions(pb) < n_transitions(pa) ? pb : pa;
    if (ph.empty()) {
      error = "phase planning failed";
      return "";
    }
    // layouts: load layout, phase layouts, store layout
    std::vector<int> plays;
    for (const Phase& f : ph) plays.push_back(add_layout(make_layout(f.S)));
    // global IO layout when a phase is not A-type: the A-type layout keeping the preferred warp bits
    int sa[5];
    for (int k = 0; k < 5; ++k) sa[k] = SB + k;
    if (__builtin_popcount(warp_pref) == WB) {
      int k = 0;
      for (int b = SB; b < TB; ++b)
        if (!((warp_pref >> b) & 1) && k < NSEL) sa[k++] = b;
    }
    if (t0free) {  // t0 + 4 group bits
      for (int k = 4; k > 0; --k) sa[k] = sa[k - 1];
      sa[0] = 0;
    }
    const int l_load = a_type(ph.front().S) ? plays.front() : add_layout(make_layout(sa));
    int l_store = a_type(ph.back().S) ? plays.back() : add_layout(make_layout(sa));
    if (d.n_remap > 0) {  // qubit remap at the store (packer's plan_remap)
      for (int t = 0; t < TB; ++t) smap[t] = slot_of_tb(t);
      for (int k = 0; k < d.n_remap; ++k) {
        const int ta = tilebit(d.remap_a[k]), tb = tilebit(d.remap_b[k]);
        if (ta < 0 || tb < 0 || (prec == 0 && (ta == 0 || tb == 0))) {
          error = "remap outside the tile";
          return "";
        }
        std::swap(smap[ta], smap[tb]);
      }
      l_store = add_layout(make_store_layout(lays[plays.back()]));
    }
    // warp-position alignment along the layout sequence: a warp bit the previous layout also has
    // keeps its warp position (a relabelling of warp indices), so a transpose synchronises only the
    // warps that exchange amplitudes -- groups of 2^(changed positions) -- and a transpose that only
    // reorders warp bits becomes warp-local
    if (!getenv("OWQS_NO_WALIGN")) {
      auto align = [&](CLayout B, const CLayout& A) {
        int nw[8];
        bool placed[8] = {}, taken[16] = {};
        for (int j = 0; j < WB; ++j) nw[j] = -1;
        for (int j = 0; j < WB; ++j)
          for (int i = 0; i < WB; ++i)
            if (B.Wb[i] == A.Wb[j]) {
              nw[j] = B.Wb[i];
              placed[j] = true;
              taken[B.Wb[i]] = true;
            }
        int k = 0;
        for (int i = 0; i < WB; ++i)
          if (!taken[B.Wb[i]]) {
            while (placed[k]) ++k;
            nw[k++] = B.Wb[i];
          }
        for (int j = 0; j < WB; ++j) B.Wb[j] = nw[j];
        return B;
      };
      int prev = l_load;
      for (int& l : plays) {
        if (l != prev) l = add_layout(align(lays[l], lays[prev]));
        prev = l;
      }
      if (l_store != prev) l_store = add_layout(align(lays[l_store], lays[prev]));
    }
    int n_trans = 0;
    {
      int cur = l_load;
      for (int l : plays) n_trans += l != cur, cur = l;
      n_trans += l_store != cur;
    }
    if (!getenv("OWQS_NO_BANKCLS")) {
      std::vector<int> used{l_load};
      for (int l : plays) used.push_back(l);
      used.push_back(l_store);
      std::sort(used.begin(), used.end());
      used.erase(std::unique(used.begin(), used.end()), used.end());
      choose_bank_classes(used);
    }
    if (coef_src == 2) o << "__constant__ owqs::PassCoef OWQS_KNAME_cp;  // the pass's decisions (graph memcpy node)\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << (32 << WB) << ", " << tile_minb() << ") OWQS_KNAME(const owqs::StepDesc d, const owqs::DevPtrs p, const owqs::PassCoef* "
      << (small ? "pc_global" : "pc") << ", const owqs::PassCoef cp) {  // pc: no __restrict__, so its loads stay behind griddepcontrol.wait\n"
      << "  (void)cp;\n"
      << "  using namespace owqs;\n"
      << "  // tile engine: width " << d.width << ", tile group slots";
    for (int j = 0; j < KHI; ++j) o << " " << gs[j];
    o << " (pass's " << d.nb_hi << "), " << d.n_ops << " ops, " << nbf << " butterflies, reduction " << red << ", "
      << ph.size() << " phase(s), " << n_trans << " transpose(s), " << iters << " tile(s) per CTA, warp bits";
    for (int j = 0; j < WB; ++j) o << " t" << lays[l_load].Wb[j];
    o << "\n";
    for (size_t f = 0; f < ph.size(); ++f) {
      o << "  // phase " << f << ": registers" << (FB ? " t0" : "");
      for (int k = 0; k < NSEL; ++k) o << " t" << ph[f].S[k];
      o << ", " << ph[f].ops.size() << " op(s)\n";
    }
    if (n_trans) o << "  extern __shared__ __align__(16) unsigned char dsm[];\n";
    if (small) {
      // grid of <= 2 waves (L2-resident states): decisions by this kernel's own prologue (every CTA,
      // warp-parallel) and the fenced last-block reduction -- one launch per pass, no decide /
      // finish kernels
      o << "  (void)pc_global;\n  __shared__ PassShared sh;\n  __shared__ PassCoef spc;\n"
        << "  pass_prologue(d, p, sh);\n"
        << "  for (int b = threadIdx.x; b < d.n_bfly; b += blockDim.x) {\n"
        << "    const double ar = sh.ka[b][0], ai = sh.ka[b][1];\n"
        << "    spc.ard[b] = ar; spc.aid[b] = ai; spc.ar[b] = (float)ar;\n"
        << "    const float fai = (float)ai;\n"
        << "    spc.B[b] = ((unsigned long long)__float_as_uint(fai) << 32) | (unsigned long long)__float_as_uint(-fai);\n"
        << "  }\n"
        << "  for (int i = threadIdx.x; i < d.n_ops; i += blockDim.x) spc.cond[i] = sh.cond[i];\n"
        << "  if (threadIdx.x == 0) spc.scale = sh.scale;\n  __syncthreads();\n"
        << "  const PassCoef* pc = &spc;\n";
    }
    o << "  __shared__ double red_s[" << (small ? 32 : 8) << "][4];\n  __shared__ int flag_s;\n"
      << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
      << "  const unsigned rk = p.rank; (void)rk; (void)d;\n"
      << "  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;\n";

    scale_pending = nbf > 0;
    if (n_trans)
      for (size_t l = 0; l < lays.size(); ++l) {
        o << "  const int sb" << l << " = (";  // byte offset
        for (int j = 0; j < 5; ++j) o << (j ? " ^ " : "") << "(((lane >> " << j << ") & 1) * " << addrb(1 << lays[l].Lb[j]) << ")";
        for (int j = 0; j < WB; ++j) o << " ^ (((warp >> " << j << ") & 1) * " << addrb(1 << lays[l].Wb[j]) << ")";
        o << ");\n";
      }
    auto wseg = [&](int l) {
      std::string e = "(0ull";
      for (int j = 0; j < WB; ++j)
        if (gslot(lays[l].Wb[j]) >= SB)
          e += " | ((unsigned long long)((warp >> " + std::to_string(j) + ") & 1) << " +
               std::to_string(gslot(lays[l].Wb[j]) - SB) + ")";
      return e + ")";
    };
    o << "  const unsigned long long wsl = " << wseg(l_load) << ";\n";
    use_smap = d.n_remap > 0;
    o << "  const unsigned long long wss = " << wseg(l_store) << ";\n";
    o << "  const int lane_st = " << lane_expr(lays[l_store], d.n_remap > 0) << ";\n";
    o << "  const int lane_ld = " << lane_expr(lays[l_load], false) << ";\n";
    use_smap = false;
    o << "  " << (prec == 0 ? "float4" : "double2") << "* __restrict__ st = reinterpret_cast<"
      << (prec == 0 ? "float4" : "double2") << "*>(p.state);\n"
      << "  for (unsigned it = 0; it < " << iters << "u; ++it) {\n"
      << "    const unsigned long long ub = (unsigned long long)blockIdx.x * " << iters << "ull + it;\n";
    emit_gb("gb0", "ub");
    // L2 prefetch of the tile the CTA one wave later (blockIdx + D, D ~ resident CTAs) will load:
    // lane m < 16 of each warp bulk-prefetches that warp's m-th 512 B segment there, so the next
    // wave's load phase hits L2 instead of waiting on HBM (OWQS_PREFETCH=D; no extra DRAM bytes)
    if (const int D = prefetch_distance(); D > 0 && iters == 1) {
      o << "    { const unsigned long long ubp = (unsigned long long)blockIdx.x + " << D << "ull;\n"
        << "    if (ubp < " << nbu << "ull && lane < 16) {\n";
      emit_gb("gbp", "ubp");
      o << "    const unsigned long long ap = 0ull";
      for (int k = 0; k < 4; ++k)
        o << " | ((lane & " << (1 << k) << ") ? " << a_seg(l_load, prec == 0 ? 2 << k : 1 << k) << "ull : 0ull)";
      o << ";\n    asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], 512;\" :: \"l\"(st + ((gbp | wsl | ap) << 5)) : \"memory\");\n"
        << "    } }\n";
    }
    // Launched with programmatic stream serialisation behind decide_kernel (or, with cached EOWQS
    // decisions, behind the previous pass): PTX guarantees the prerequisite grid's stores only
    // after griddepcontrol.wait, so every read of the state (and of PassCoef) comes after it. Before
    // the wait, lane m < 16 of each warp bulk-prefetches its m-th 512 B load segment into L2 -- L2
    // is the point of coherence, so a prefetched line can never be older than the writer's store
    // (off by default, OWQS_PDL_PREFETCH=1).
    if (!small) {
      if (pdl_prefetch()) {
        o << "    if (lane < 16) {\n      const unsigned long long ap = 0ull";
        for (int k = 0; k < 4; ++k)
          o << " | ((lane & " << (1 << k) << ") ? " << a_seg(l_load, prec == 0 ? 2 << k : 1 << k) << "ull : 0ull)";
        o << ";\n      asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], 512;\" :: \"l\"(st + ((gb0 | wsl | ap) << 5)) : \"memory\");\n    }\n";
      }
      o << "    asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
    }
    if (prec == 0)
      for (int q = 0; q < P; q += 2)
        o << "    u64 x" << q << ", x" << q + 1 << "; { const float4 w = __ldcs(st + (((gb0 | wsl | " << a_seg(l_load, q)
          << "ull) << 5) + lane_ld)); x" << q << " = pk(w.x, w.y); x" << q + 1 << " = pk(w.z, w.w); }\n";
    else
      for (int q = 0; q < P; ++q)
        o << "    double xr" << q << ", xi" << q << "; { const double2 w = __ldcs(st + (((gb0 | wsl | " << a_seg(l_load, q)
          << "ull) << 5) + lane_ld)); xr" << q << " = w.x; xi" << q << " = w.y; }\n";
    if (nbf > 0 && prec == 0) o << "    const float sck = (float)" << PC << "scale;\n    const u64 scale = bc(sck); (void)scale;\n";
    if (nbf > 0 && prec == 1) o << "    const double sck = " << PC << "scale;\n    const double scale = sck; (void)scale;\n";
    lay = l_load;
    for (int q = 0; q < P; ++q) perm[q] = q;
    std::vector<int> bidx(d.n_ops, -1);
    {
      int bi = 0;
      for (int i = 0; i < d.n_ops; ++i)
        if (d.ops[i].type == OP_BFLY) bidx[i] = bi++;
    }
    int left = n_trans;
    for (size_t f = 0; f < ph.size(); ++f) {
      if (plays[f] != lay) emit_tile_transition(plays[f], --left == 0);
      o << "    // ---- phase " << f << "\n";
      for (int i : ph[f].ops) {
        if (i == n_ops_) {  // the reduction (after every op)
          flush();
          emit_scale(nbf);
          reduce();
        } else {
          emit_op(i, bidx[i]);
        }
      }
    }
    if (l_store != lay) emit_tile_transition(l_store, --left == 0);
    use_smap = d.n_remap > 0;
    if (d.n_ops > 0 && prec == 0)
      for (int q = 0; q < P; q += 2)
        o << "    __stcs(st + (((gb0 | wss | " << a_seg(l_store, q) << "ull) << 5) + lane_st), make_float4(lo(" << X(q)
          << "), hi(" << X(q) << "), lo(" << X(q + 1) << "), hi(" << X(q + 1) << ")));\n";
    if (d.n_ops > 0 && prec == 1)
      for (int q = 0; q < P; ++q)
        o << "    __stcs(st + (((gb0 | wss | " << a_seg(l_store, q) << "ull) << 5) + lane_st), make_double2(" << XR(q)
          << ", " << XI(q) << "));\n";
    use_smap = false;
    o << "  }\n";
    if (nred > 0)
      o << "  double acc[4] = {acc0, acc1, acc2, acc3};\n"
        << (small ? "  reduce_finish_grid<" : "  block_partial<") << nred
        << (small ? ">(acc, p, red_s, &flag_s);\n" : ">(acc, p, red_s);  // grid_finish_kernel sums\n");
    o << "}\n";
    return o.str();
  }

  std::string run() { return tile ? run_tile() : run_direct(); }
};

// ---- compile cache ------------------------------------------------------------------------------
struct CacheEntry {
  std::shared_ptr<JitModule> mod;
};
std::mutex g_mu;
std::unordered_map<std::string, std::shared_ptr<JitModule>> g_cache;  // kernel name -> module

// NVRTC of the toolkit the library was built with, loaded by absolute path into its own symbol scope
// (RTLD_LOCAL | RTLD_DEEPBIND). Linking -lnvrtc would bind to whichever libnvrtc.so.12 the process
// loaded first -- after `import torch` that is torch's bundled cu128 copy, whose back end emits
// measurably slower sm_100a code for the same source (C3 pass kernels: 62.5 vs 50.5 ms per run).
struct Nvrtc {
  void* h = nullptr;
  std::string err;
  int major = 0, minor = 0;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*errstr)(nvrtcResult) = nullptr;
  nvrtcResult (*version)(int*, int*) = nullptr;
};

const Nvrtc& nvrtc() {
  static const Nvrtc n = [] {
    Nvrtc x;
    const char* path = getenv("OWQS_NVRTC");
#ifdef OWQS_NVRTC_PATH
    if (!path) path = OWQS_NVRTC_PATH;
#endif
    if (!path) path = "libnvrtc.so.12";
    x.h = dlopen(path, RTLD_NOW | RTLD_LOCAL | RTLD_DEEPBIND);
    if (!x.h) {
      const char* e = dlerror();
      x.err = std::string("cannot load NVRTC from ") + path + ": " + (e ? e : "?");
      return x;
    }
    bool ok = true;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(x.h, name));
      if (!f) ok = false;
    };
    sym(x.create, "nvrtcCreateProgram");
    sym(x.compile, "nvrtcCompileProgram");
    sym(x.log_size, "nvrtcGetProgramLogSize");
    sym(x.log, "nvrtcGetProgramLog");
    sym(x.cubin_size, "nvrtcGetCUBINSize");
    sym(x.cubin, "nvrtcGetCUBIN");
    sym(x.destroy, "nvrtcDestroyProgram");
    sym(x.errstr, "nvrtcGetErrorString");
    sym(x.version, "nvrtcVersion");
    if (!ok) {
      x.err = std::string("NVRTC at ") + path + " lacks an entry point";
      return x;
    }
    x.version(&x.major, &x.minor);
    return x;
  }();
  return n;
}

std::string compile_tu(const std::string& src, std::vector<char>& cubin) {
  const Nvrtc& nv = nvrtc();
  if (!nv.err.empty()) return nv.err;
  nvrtcProgram prog;
  nvrtcResult r = nv.create(&prog, src.c_str(), "owqs_pass_jit.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return std::string("nvrtcCreateProgram: ") + nv.errstr(r);
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DOWQS_JIT=1"};
  // ptxas options (OWQS_PTXAS, e.g. "-O1"; default: ptxas' own -O3). Found on C3's heavy passes:
  // with the own-tile L2 prefetch (asm volatile, memory clobber) ahead of griddepcontrol.wait, -O3
  // rematerialised every coefficient load per use (582 LDCU, 3152 instructions = 50 KB of SASS,
  // instruction-cache hit rate 63 %, "no instruction" 46 % of the warp-stall samples); -O1 kept 49
  // LDCU / 2632 instructions (C3 37.6 -> 36.0 ms). Without that prefetch (now off by default) -O1
  // and -O3 emit the same SASS for C3's tile kernels (tools/jit_dump.py + cuobjdump), and -O3 is
  // 2 % faster on C4's several-tiles-per-CTA kernels (793 vs 811 ms).
  static const std::string ptxas = [] {
    const char* e = getenv("OWQS_PTXAS");
    return std::string(e && strcmp(e, "default") ? e : "");
  }();
  const std::string ptxas_opt = "--ptxas-options=" + ptxas;
  if (!ptxas.empty()) opts.push_back(ptxas_opt.c_str());
  r = nv.compile(prog, (int)opts.size(), opts.data());
  std::string err;
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv.log(prog, &log[0]);
    err = std::string("nvrtcCompileProgram: ") + nv.errstr(r) + "\n" + log;
  } else {
    size_t n = 0;
    nv.cubin_size(prog, &n);
    cubin.resize(n);
    nv.cubin(prog, cubin.data());
  }
  nv.destroy(&prog);
  return err;
}

}  // namespace

std::string jit_nvrtc_version(int* major, int* minor) {
  const Nvrtc& nv = nvrtc();
  *major = nv.major;
  *minor = nv.minor;
  return nv.err;
}

int jit_engine(const StepDesc& d, int prec) {
  if (d.kind != ST_PASS) return 0;
  if (d.width >= tile_bits(prec) && d.nb_hi <= tile_g(prec) && !getenv("OWQS_JIT_NO_TILE")) return 2;
  if (d.nb_hi > KMAX_AOT) return -1;  // needs the tile engine
  const int SB = prec == 0 ? 6 : 5;
  const int unr = jit_unr_of(d.nb_hi);
  const int slack = d.width - SB - d.nb_hi - (unr == 4 ? 2 : (unr == 2 ? 1 : 0)) - 3;
  return slack >= 0 ? 1 : 0;
}

bool jit_eligible(const StepDesc& d, int prec) { return jit_engine(d, prec) > 0; }

int jit_max_group(int prec, bool no_jit) {
  return (!no_jit && !getenv("OWQS_JIT_NO_TILE")) ? tile_g(prec) : KMAX_AOT;
}

int jit_smem_carveout(int engine, int prec) {
  if (engine != 2) return -1;  // cudaSharedmemCarveoutDefault
  if (const char* e = getenv("OWQS_CARVEOUT")) return atoi(e);
  // CTAs per SM (register-limited) x (tile + static + reserved), as a percentage of 228 KB
  // (static: red_s[8][4] + flag; reserved: 1 KB per CTA) -- 3 x 64 KB tiles fit the 196 KB split
  const int per = jit_dyn_smem(2, prec) + 288 + 1024;
  const int ctas = Gen::tile_minb_for(prec);
  return std::min(100, (ctas * per * 100 + 233471) / 233472);
}

int jit_block_threads(int engine, int prec) {
  if (engine != 2) return 256;
  return prec == 0 ? (32 << tile_geom().wb) : (32 << (tile_g(1) - 4));
}

bool jit_tile_small(const StepDesc& d, int prec) {
  if (jit_engine(d, prec) != 2) return false;
  static const unsigned lim = [] {
    const char* e = getenv("OWQS_TILE_SMALL_MAX");
    // default off: measured on C2 (QFT-20, 128 CTAs per pass) the per-CTA prologue is slower than
    // one decide_kernel overlapped by programmatic dependent launch (0.912 vs 0.869 ms per run)
    return e ? (unsigned)atoi(e) : 0u;
  }();
  return jit_tile_blocks(d, prec) <= lim;
}

unsigned jit_tile_blocks(const StepDesc& d, int prec) {
  const uint64_t nbu = 1ull << (d.width - tile_bits(prec));
  // test hook OWQS_TILE_MAX_BLOCKS (power of two): cap the grid lower than RED_MAX_BLOCKS so that
  // small states exercise the several-tiles-per-CTA path of states above 2^20 tiles
  static const uint64_t cap = [] {
    const char* e = getenv("OWQS_TILE_MAX_BLOCKS");
    const uint64_t v = e ? (uint64_t)atoll(e) : 0;
    return (v && !(v & (v - 1)) && v < (uint64_t)RED_MAX_BLOCKS) ? v : (uint64_t)RED_MAX_BLOCKS;
  }();
  return (unsigned)(nbu > cap ? cap : nbu);
}

int jit_dyn_smem(int engine, int prec) {
  return engine == 2 ? 16 << (tile_bits(prec) - (prec == 0 ? 1 : 0)) : 0;  // one 16 B unit per pair / amplitude
}

const std::string& jit_prelude() {
  static const std::string s = std::string(kPreludeInternal) + "\n" + kPreludeCommon + "\n" + kHelpers;
  return s;
}

namespace {
int count_of(const std::string& s, const char* what) {
  int n = 0;
  for (size_t i = s.find(what); i != std::string::npos; i = s.find(what, i + 1)) ++n;
  return n;
}
int transposes_of(const std::string& s) {
  const size_t i = s.find(" transpose(s)");
  if (i == std::string::npos) return 0;
  size_t j = i;
  while (j > 0 && isdigit((unsigned char)s[j - 1])) --j;
  return atoi(s.c_str() + j);
}
}  // namespace

std::string jit_pass_source(const StepDesc& d, int prec, std::string* name, int coef_src) {
  const int eng = jit_engine(d, prec);
  if (!eng) return "";
  if (eng != 2 || jit_tile_small(d, prec)) coef_src = 0;
  Gen g(d, prec, eng == 2, false, coef_src);
  if (!g.error.empty()) return "";
  std::string body = g.run();
  if (!g.error.empty()) return "";
  // complex64 tile passes: the t0-free plan (phases over any 5 of the 13 tile bits) where it needs
  // fewer transposes and no more shared-memory instructions (8 B accesses when t0 is a lane bit);
  // OWQS_T0_FREE=0 / 1 forces it off / on for every pass
  const char* tf = getenv("OWQS_T0_FREE");
  if (eng == 2 && prec == 0 && !(tf && atoi(tf) == 0)) {
    Gen g2(d, prec, true, true, coef_src);
    std::string b2 = g2.error.empty() ? g2.run() : std::string();
    if (g2.error.empty() && !b2.empty()) {
      const int smem1 = count_of(body, "reinterpret_cast<"), smem2 = count_of(b2, "reinterpret_cast<");
      if ((tf && atoi(tf) == 1) || (transposes_of(b2) < transposes_of(body) && smem2 <= smem1)) body = b2;
    }
  }
  const std::string nm = std::string(eng == 2 ? "owqs_tile_" : "owqs_pass_") + (prec == 0 ? "c64_" : "c128_") + hex64(fnv1a(body));
  const std::string key = "OWQS_KNAME";
  for (size_t at = body.find(key); at != std::string::npos; at = body.find(key, at + nm.size())) body.replace(at, key.size(), nm);
  if (name) *name = nm;
  return body;
}

std::string jit_compile(const std::vector<std::string>& names, const std::vector<std::string>& sources,
                        std::vector<JitModule>& out, double* compile_ms) {
  auto t0 = std::chrono::steady_clock::now();
  out.clear();
  // dedupe; split into cached / to compile
  std::vector<int> todo;
  std::map<std::string, int> seen;
  std::vector<std::shared_ptr<JitModule>> mods;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < names.size(); ++i) {
      if (seen.count(names[i])) continue;
      seen[names[i]] = (int)i;
      auto it = g_cache.find(names[i]);
      if (it != g_cache.end()) {
        if (std::find(mods.begin(), mods.end(), it->second) == mods.end()) mods.push_back(it->second);
      } else {
        todo.push_back((int)i);
      }
    }
  }
  if (!todo.empty()) {
    const int per_tu = 6;
    const int n_tu = ((int)todo.size() + per_tu - 1) / per_tu;
    std::vector<std::shared_ptr<JitModule>> fresh(n_tu);
    std::vector<std::string> errs(n_tu);
    int n_thr = (int)std::thread::hardware_concurrency();
    n_thr = std::max(1, std::min(n_thr, std::min(n_tu, 32)));
    std::mutex qm;
    int next = 0;
    auto worker = [&]() {
      while (true) {
        int k;
        {
          std::lock_guard<std::mutex> lk(qm);
          if (next >= n_tu) return;
          k = next++;
        }
        auto m = std::make_shared<JitModule>();
        std::string src = jit_prelude();
        for (int j = k * per_tu; j < std::min((int)todo.size(), (k + 1) * per_tu); ++j) {
          src += "\n" + sources[todo[j]];
          m->names.push_back(names[todo[j]]);
        }
        errs[k] = compile_tu(src, m->cubin);
        fresh[k] = m;
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < n_thr; ++t) th.emplace_back(worker);
    for (auto& t : th) t.join();
    for (int k = 0; k < n_tu; ++k)
      if (!errs[k].empty()) return errs[k];
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& m : fresh) {
      for (auto& n : m->names) g_cache[n] = m;
      mods.push_back(m);
    }
  }
  for (auto& m : mods) out.push_back(*m);
  if (compile_ms) *compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return "";
}

size_t jit_coef_param_offset(cudaKernel_t k) {
  size_t off = 0, size = 0;
  if (cudaFuncGetParamInfo((const void*)k, 3, &off, &size) != cudaSuccess || size != sizeof(PassCoef)) {
    cudaGetLastError();
    return (size_t)-1;
  }
  return off;
}

cudaError_t jit_launch(cudaKernel_t k, int max_blocks, const StepDesc& d, const DevPtrs& p, const PassCoef* pc, int prec,
                       cudaStream_t s, const PassCoef* cp_host, cudaGraphDeviceNode_t* dev_node, bool no_pdl) {
  const int eng = jit_engine(d, prec);
  const int SB = prec == 0 ? 6 : 5;
  const int unr = jit_unr_of(d.nb_hi);
  StepDesc dd = d;
  DevPtrs pp = p;
  const PassCoef* pcc = pc;
  if (eng == 2) {  // non-persistent: one CTA per tile (or iters tiles above RED_MAX_BLOCKS)
    static const PassCoef zero{};
    PassCoef cp = cp_host ? *cp_host : zero;
    const uint64_t blocks = jit_tile_blocks(d, prec);  // the generator's tiles-per-CTA use the same count
    void* args[] = {&dd, &pp, &pcc, &cp};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(jit_block_threads(eng, prec));
    cfg.dynamicSmemBytes = (size_t)jit_dyn_smem(eng, prec);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (no_pdl || getenv("OWQS_NO_PDL") || jit_tile_small(d, prec)) ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (dev_node) {  // captured launch whose PassCoef parameter decide_kernel rewrites every run
      attr[1].id = cudaLaunchAttributeDeviceUpdatableKernelNode;
      attr[1].val.deviceUpdatableKernelNode.deviceUpdatable = 1;
      attr[1].val.deviceUpdatableKernelNode.devNode = nullptr;
      cfg.numAttrs = 2;
    }
    const cudaError_t e = cudaLaunchKernelExC(&cfg, (const void*)k, args);
    if (dev_node) *dev_node = attr[1].val.deviceUpdatableKernelNode.devNode;
    return e;
  }
  const int slack = d.width - SB - d.nb_hi - (unr == 4 ? 2 : (unr == 2 ? 1 : 0)) - 3;
  const uint64_t blocks = std::min<uint64_t>(1ull << slack, (uint64_t)std::max(1, max_blocks));
  void* args[] = {&dd, &pp};
  return cudaLaunchKernel((const void*)k, dim3((unsigned)blocks), dim3(256), args,
                          (size_t)jit_dyn_smem(eng, prec), s);
}

}  // namespace owqs
