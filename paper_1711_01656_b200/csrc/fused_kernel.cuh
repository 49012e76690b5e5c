// Fused integral histogram + sliding-window matcher (one pass over the frame).
//
// Replaces build_integral_histogram followed by hist_distance_map (reference
// integral.cpp:548-551, likelihood.cpp:193-225) without re-reading the tensor: the
// window counts come from a vertical running histogram kept in shared memory.
//
// CTA = (128-column strip, band of rows, group of <= 128 bins); 8 warps x 16 bins.
//   * V part (optional, `STORE`): the build sweep of sweep_common.cuh writes the
//     integral-histogram rows of the strip (same bits as spct_cu_ih_build).
//   * vc: for each of the CTA's bins and each of 256 "extended" columns
//     [x0-128, x0+128) the count of that bin in the column over the last kh rows
//     (u16 cells, two per 32-bit word, 64 KB).  Every row, thread t adds the entering
//     pixel of column t and removes the pixel that left the window: two shared
//     atomics per column, independent of the bin count.
//   * G: per bin, the inclusive prefix of vc along the 256 columns (u16 pairs, lane l
//     owns columns 4l..4l+3 of each half; in-lane IMAD prefix + one 16-bit-packed warp
//     scan).  The count of the kw x kh window whose bottom-right pixel is (e, y) is
//     G(e) - G(e - kw), read back through a per-warp staging row.
//   * distance: Minkowski p = 1 / intersection with an integral template
//     (s_k = T t_k in Z, the template-crop case) is exact integer arithmetic:
//     sum_k |c_k - s_k| = C + S - 2 sum_k min(c_k, s_k), with min.u16x2 on packed
//     pairs.  Every other metric / p evaluates likelihood.cpp's per-bin term in FP64.
//   * the 8 warps' per-window partials are combined in a fixed order through shared
//     memory and written as one partial-map row (float64) per CTA row.
#pragma once

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "spct_internal.h"
#include "sweep_common.cuh"

namespace spct_fused {

using namespace spct_dev;
using namespace spct_impl;

constexpr int kB = 16;
constexpr int kGroupBins = 128;          // bins per launch group (the widest CTA: 8 warps x 16)
constexpr int kExt = 256;                // extended columns per CTA (128 halo + 128 strip)
constexpr int kVcWords = kExt / 2;       // u16 pairs per bin row
constexpr int kVcStride = kVcWords + kVcWords / 8;  // row stride: 4 padding words after every 32

struct FusedParams {
    int kw, kh, nu, nv;
    int metric, p_kind, T_pow2, accumulate;
    double p, T, invT;
    int group0;                  // first slab-local bin of this launch's bin group
    const double* tmpl;          // full template, indexed by global bin
    const uint32_t* prep;        // [0] path kind (0 FP64, 1 integral template, 2 fractional), [1..] srep (slab-local)
    const long long* S_group;    // sum of floor(s_k) per 128-bin group
    const double* Sr_group;      // sum of the fractional parts r_k = s_k - floor(s_k) per 128-bin group
    const double* rfrac;         // r_k per slab-local bin (kind 2)
    const float4* c3;            // kind 3, per slab-local bin: {64 floor(s_k) + 2 R_k (int bits), r_k - R_k / 32,
                                 //   sqrt(t_k / T), s_k}, R_k = rint(32 r_k)
    const double2* c3slab;       // kind 3, per 16-bin slab: {sum s_k^2, sum s_k}
    double* partial;
    double* map;                 // non-null: write the finished likelihood map (one group = every bin)
    double inv_p, dmax, inv_dmax;  // inv_dmax != 0 iff dmax is a power of two (exact product)
    int W, H;
    int frac;     // host: the fractional variant is launched instead of the FP64 one
    int path;     // host: 1 = integer metric (MODE 1 + MODE 2 or 0), 3 / 4 / 0 = that MODE only
    int fp_kind;  // FP64 path term: 0 Minkowski p=1, 1 p=2, 2 general p, 3 intersection, 4 Bhattacharyya, 5 chi-square
};

// likelihood.cpp:220-221 (and the extension metrics), as in hist_match.cu finalize_kernel.
__device__ __forceinline__ double finalize_L(double s, const FusedParams& f) {
    double L;
    if (f.metric == SPCT_METRIC_MINKOWSKI) {
        const double d = f.p_kind == 1 ? s : pow(s, f.inv_p);
        L = __dsub_rn(1.0, f.inv_dmax != 0.0 ? __dmul_rn(d, f.inv_dmax) : __ddiv_rn(d, f.dmax));
    } else if (f.metric == SPCT_METRIC_CHISQ) {
        L = __dsub_rn(1.0, __dmul_rn(s, 0.5));  // == s / 2 exactly
    } else {
        L = s;
    }
    return L < 0.0 ? 0.0 : (L > 1.0 ? 1.0 : L);
}

__device__ __forceinline__ uint32_t min_u16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

__device__ __forceinline__ uint32_t min_s16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// pow for a general Minkowski order, kept out of line (inlined at every call site it
// bloats the sweep past the instruction cache).
static __device__ __noinline__ double pow_term(double a, double p) { return pow(a, p); }

// Per-bin term of the general path (same arithmetic as hist_match.cu bin_term).
__device__ __forceinline__ double general_term(uint32_t c, double t, const FusedParams& f) {
    const double cd = static_cast<double>(c);
    const double q = f.T_pow2 ? __dmul_rn(cd, f.invT) : __ddiv_rn(cd, f.T);
    switch (f.metric) {
        case SPCT_METRIC_MINKOWSKI: {
            const double a = fabs(__dsub_rn(q, t));
            if (f.p_kind == 1) return a;
            if (f.p_kind == 2) return __dmul_rn(a, a);
            return pow_term(a, f.p);
        }
        case SPCT_METRIC_INTERSECTION:
            return fmin(q, t);
        case SPCT_METRIC_BHATTACHARYYA:
            return sqrt(__dmul_rn(q, t));
        default: {
            const double den = __dadd_rn(q, t);
            if (!(den > 0.0)) return 0.0;
            const double df = __dsub_rn(q, t);
            return __ddiv_rn(__dmul_rn(df, df), den);
        }
    }
}


// vc rows are padded: word w of a bin row lives at w + 4 (w >> 5), so the quarter-warp
// reads of 8 consecutive words per lane (two 16-B loads, 8 lanes per phase) hit 8
// distinct bank groups, and every quad the integer path reads sits at a fixed offset
// from the lane's strip quad.
__device__ __forceinline__ int vcw(int w) { return w + ((w >> 3) & ~3); }

// FP64 path term of one window count, specialised per metric (FusedParams::fp_kind) so
// the hot loop carries only its own arithmetic (likelihood.cpp:215-219 and the thesis
// metrics).  q = c * (1 / T): within an ulp of the reference's division, inside the
// fused path's tolerance.
template <int FK>
__device__ __forceinline__ double fp_term(uint32_t c, double t, double invT, double p) {
    const double q = __dmul_rn(static_cast<double>(c), invT);
    if (FK == 0) return fabs(__dsub_rn(q, t));
    if (FK == 1) {
        const double a = __dsub_rn(q, t);
        return __dmul_rn(a, a);
    }
    if (FK == 2) return pow_term(fabs(__dsub_rn(q, t)), p);
    if (FK == 3) return fmin(q, t);
    if (FK == 4) return sqrt(__dmul_rn(q, t));
    const double den = __dadd_rn(q, t);
    if (!(den > 0.0)) return 0.0;
    const double df = __dsub_rn(q, t);
    return __ddiv_rn(__dmul_rn(df, df), den);
}

// u16 count -> float, exactly (c < 2^23): 2^23 + c by bit pattern, minus 2^23.
__device__ __forceinline__ float count_f32(uint32_t c) { return __int_as_float(0x4B000000u | c) - 8388608.0f; }

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// MODE 3 per-bin terms of one window count c (cst = FusedParams::c3 of the bin):
//   FK 1 (p = 2): T^2 d^2 = sum (c - s)^2 = (1/32) sum c (32 c - 64 f - 2 R) - 2 sum c r_lo + sum s^2
//     with s = f + R/32 + r_lo: the first sum exact in int32 (|.| < 2^31 for kw kh <= 4096), the
//     second (|r_lo| <= 1/64) in FP32, so no cancellation is left in FP32 near d = 0;
//   FK 4 (Bhattacharyya): sum sqrt(q t) = sum sqrt(c) sqrt(t / T), FP32 (non-negative terms);
//   FK 5 (chi-square): (q - t)^2 / (q + t) = q + t - 4 q t / (q + t): FP32 sum of
//     Y = sum c s / (c + s) (non-negative terms); the linear part is exact (window counts).
template <int FK>
__device__ __forceinline__ void f32_term(uint32_t c, const float4& cst, int& ai, float& af) {
    const float cf = count_f32(c);
    if (FK == 1) {
        const int ci = static_cast<int>(c);
        ai += ci * (32 * ci - __float_as_int(cst.x));
        af = fmaf(cf, cst.y, af);
    } else if (FK == 4) {
        af = fmaf(sqrt_approx(cf), cst.z, af);
    } else {
        af = fmaf(cf * cst.w, rcp_approx(cf + cst.w), af);
    }
}

// Window counts (general path), phase 1: for bin row `vrow`, the inclusive prefix G of the
// 256 extended columns for the lane's 8 columns (u16 pairs): the halo half (a0, a1) and
// the strip half (b0, b1); with STAGE they are also written to `g` (the warp's staging
// row for this bin) for the general-kw partner reads.
template <bool STAGE>
__device__ __forceinline__ void window_prefix(const uint32_t* vrow, uint32_t* g, int lane, uint32_t& a0, uint32_t& a1,
                                              uint32_t& b0, uint32_t& b1) {
    const uint2 wa = *reinterpret_cast<const uint2*>(vrow + vcw(2 * lane));
    const uint2 wb = *reinterpret_cast<const uint2*>(vrow + vcw(64 + 2 * lane));
    a0 = wa.x * 0x10001u;
    a1 = wa.y * 0x10001u + __byte_perm(a0, 0, 0x3232);
    b0 = wb.x * 0x10001u;
    b1 = wb.y * 0x10001u + __byte_perm(b0, 0, 0x3232);
    const uint32_t tot = __byte_perm(a1, b1, 0x7632);  // {sum a, sum b}
    const uint32_t inc = warp_incl_scan(tot);
    const uint32_t ex = inc - tot;
    const uint32_t T1 = __byte_perm(__shfl_sync(0xffffffffu, inc, 31), 0, 0x1010);  // total of the halo half
    const uint32_t ba = __byte_perm(ex, 0, 0x1010);
    const uint32_t bb = __byte_perm(ex, 0, 0x3232) + T1;
    a0 += ba;
    a1 += ba;
    b0 += bb;
    b1 += bb;
    if (STAGE) {
        *reinterpret_cast<uint2*>(g + 2 * lane) = make_uint2(a0, a1);
        *reinterpret_cast<uint2*>(g + 64 + 2 * lane) = make_uint2(b0, b1);
    }
}

// Window counts (general path), phase 2 (after a __syncwarp): c = G(e) - G(e - kw) for the
// lane's four windows, as two u16 pairs {j=0, j=1}, {j=2, j=3}.
__device__ __forceinline__ void window_diff(const uint32_t* g, int pw, int psh, uint32_t b0, uint32_t b1,
                                            uint32_t& c0, uint32_t& c1) {
    const uint32_t q0 = g[pw], q1 = g[pw + 1], q2 = g[pw + 2];
    c0 = b0 - __funnelshift_r(q0, q1, psh);
    c1 = b1 - __funnelshift_r(q1, q2, psh);
}

// Inclusive scan step over 8-lane segments (shuffle in-range predicate, no select).
__device__ __forceinline__ uint32_t scan_add8(uint32_t v, int o) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
        "shfl.sync.up.b32 t|p, %1, %2, 0x1800, 0xffffffff;\n\t"
        "@p add.u32 %1, %1, t;\n\t"
        "mov.u32 %0, %1;\n\t}"
        : "=r"(r), "+r"(v)
        : "r"(o));
    return r;
}

// Window counts (integer path), quarter-warp layout: lane m (0..7) of a quarter owns the 16
// windows ending at strip columns 16m .. 16m+15 (extended columns e = 128 + 16m + i) of one
// bin.  With vc the bin's running column counts over the last kh rows,
//     c(e) = c(127) + sum_{x=128..e} delta(x),   delta(x) = vc(x) - vc(x - kw),
// and the anchor c(127) = sum of vc over [128 - kw, 128), i.e. of the lane's vc(e - kw)
// values with 16m + i < kw.  The in-lane prefix starts at +4080 (= 16 * 255 >= any
// negative partial sum), so every prefix half is a non-negative u16 and the broadcast of
// a word's high half is exact; the same offset per lane is removed once, with the anchor,
// where the true counts 0 <= c <= kw*kh < 2^16 make the packed pairs exact.  One 8-lane
// scan of {anchor partial, lane prefix total} per bin: 3 shuffle steps + 1 broadcast.
// Result: the window counts c(16m + 2j + h) = w[j].half(h) + off, with w[j] packed u16 pairs
// in [0, 8160] and `off` the lane's (signed) offset.
// pb: the lane's strip quad (word 64 + 8m, padded); the vc(e - kw) quads of kw = 64 / 128
// are at fixed offsets from it; the general kw reads 9 words from `vrow`.
template <int KWM>
__device__ __forceinline__ void window_counts_q(const uint32_t* pb, const uint32_t* vrow, int m, int aw0, int apsh,
                                                const uint32_t* amask, uint32_t (&w)[8], int& off) {
    uint32_t b[8], a[8];
    {
        const uint4 x = *reinterpret_cast<const uint4*>(pb), y = *reinterpret_cast<const uint4*>(pb + 4);
        b[0] = x.x, b[1] = x.y, b[2] = x.z, b[3] = x.w, b[4] = y.x, b[5] = y.y, b[6] = y.z, b[7] = y.w;
    }
    if (KWM == 64 || KWM == 128) {
        const uint32_t* pa = pb - (KWM == 64 ? 36 : 72);
        const uint4 x = *reinterpret_cast<const uint4*>(pa), y = *reinterpret_cast<const uint4*>(pa + 4);
        a[0] = x.x, a[1] = x.y, a[2] = x.z, a[3] = x.w, a[4] = y.x, a[5] = y.y, a[6] = y.z, a[7] = y.w;
    } else {
        uint32_t r[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) r[i] = vrow[vcw(aw0 + i)];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __funnelshift_r(r[j], r[j + 1], apsh);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // two independent 4-word chains, joined below
        const uint32_t d = b[j] - a[j];  // {delta, delta} pair, linear encoding
        w[j] = d * 0x10001u + ((j & 3) ? __byte_perm(w[j - 1], 0, 0x3232) : 0x0FF00FF0u);
    }
    {   // words 4..7 started from the same +4080 offset: add the first half's total
        const uint32_t join = (w[3] >> 16) - 4080u;  // >= -4080: the halves stay non-negative
        const uint32_t j2 = join * 0x10001u;
#pragma unroll
        for (int j = 4; j < 8; ++j) w[j] += j2;
    }
    uint32_t x;  // anchor partial as a u16 pair sum
    if (KWM == 64 || KWM == 128) {
        x = (a[0] + a[1]) + (a[2] + a[3]) + (a[4] + a[5]) + (a[6] + a[7]);
        if (KWM == 64) x = m < 4 ? x : 0u;
    } else {
        const uint4 m0 = *reinterpret_cast<const uint4*>(amask + 8 * m);
        const uint4 m1 = *reinterpret_cast<const uint4*>(amask + 8 * m + 4);
        x = ((a[0] & m0.x) + (a[1] & m0.y)) + ((a[2] & m0.z) + (a[3] & m0.w)) + ((a[4] & m1.x) + (a[5] & m1.y)) +
            ((a[6] & m1.z) + (a[7] & m1.w));
    }
    const uint32_t pack = ((x + (x >> 16)) & 0xFFFFu) | (w[7] & 0xFFFF0000u);  // {anchor partial, prefix total}
    uint32_t inc = pack;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) inc = scan_add8(inc, o);
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 7, 8);
    off = static_cast<int>((tot & 0xFFFFu) + ((inc - pack) >> 16)) - 4080 * (m + 1);
}

// Cross-quarter reduce-scatter of 8 packed words: afterwards lane (q, m) holds in v[0..1]
// the warp's sums of words 4 (q >> 1) + 2 (q & 1) + {0, 1}.
__device__ __forceinline__ void quarter_reduce(uint32_t (&v)[8], int q) {
    const bool hi2 = q & 2, hi1 = q & 1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t send = hi2 ? v[j] : v[j + 4];
        const uint32_t keep = hi2 ? v[j + 4] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const uint32_t send = hi1 ? v[j] : v[j + 2];
        const uint32_t keep = hi1 ? v[j + 2] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
}

// Geometry of a CTA with S strips side by side (S * 128 columns of windows) and NWB =
// 8 / S warps per strip (16 NWB bins).  Narrow histograms (16 NWB bins <= 64) use several
// strips per CTA, so every CTA has 8 warps and the 128-column halo of staged columns (the
// kw - 1 columns left of the first window) is shared by S strips instead of one.
template <int S>
struct Geo {
    static constexpr int NW = 8;                      // warps per CTA
    static constexpr int NWB = NW / S;                // warps (16-bin slabs) per strip
    static constexpr int NB = NWB * kB;               // bins per CTA
    static constexpr int NT = 32 * NW;                // threads per CTA
    static constexpr int E = kStrip * (S + 1);        // staged ("extended") columns
    static constexpr int VW = E / 2;                  // u16-pair words per bin row of vc
    static constexpr int VS = VW + VW / 8;            // padded row stride (4 words per 32)
    static constexpr int CPT = (E + NT - 1) / NT;     // staged columns per thread
    static constexpr int WOFF = kVcWords / 2 + kVcWords / 16;  // padded vc words per strip (72)
};

// ALLB (integer path only): the CTA's bin group is the whole histogram, so the window
// total over the group's bins is kw * kh and need not be accumulated.
// SK (source kind of the staging loads): 1 = 8-bit gray with the default range
// (bin = v * nbins >> 8), 2 = a uint16 BinMap (bin = v), 0 = the generic per-kind dispatch,
// 3 = SK 1 with 4-byte aligned rows, staged four columns per thread (4- and 8-strip CTAs).
// S: strips per CTA (Geo<S>); 1 for >= 65 bins, 2 / 4 / 8 for <= 64 / 32 / 16 bins.
template <int S>
constexpr size_t smem_bytes_s() {
    using G = Geo<S>;
    return (size_t(G::NB + 1) * G::VS + size_t(G::NW) * 4 * kVcWords + G::NB + 2 * S * G::NB + 64) * 4 +
           size_t(2) * G::NW * kStrip * 8 + size_t(2) * kStrip * S * 2;
}

// MODE: 0 = the FP64 per-bin path (any metric), 1 = the exact integer path (integral
// template, p = 1 / intersection), 2 = the integer path on floor(s_k) plus the fractional
// correction sum_{k: c_k > floor(s_k)} r_k (any template, p = 1 / intersection, kw kh <= 4096),
// 3 = the full-warp layout of MODE 0 with integer / FP32 per-bin terms for p = 2 (kw kh <= 4096)
// (f32_term below), 4 / 5 = Bhattacharyya / chi-square in the quarter layout of the integer
// paths: per window and bin sqrt(c) sqrt(t / T), resp. c s / (c + s) (chi-square through
// (q - t)^2 / (q + t) = q + t - 4 q t / (q + t)), in FP32 (16 windows per lane, four bins per
// lane, the quarters summed in a fixed order), the warps' partials combined in FP64;
// 6 = p = 2 in the quarter layout: MODE 3's exact int32 part c (32 c - X) and FP32 part c Y
// per window and bin (kw kh <= 4096).
template <bool STORE, int MODE, int KWM, bool ALLB, int SK, int S>
__global__ void __launch_bounds__(256, 2) sweep_match_kernel(QuantParams q, PixelMode pm, spct_ih out, int Lb, int Wp,
                                                             int band_rows, int nstrips, FusedCarries fc,
                                                             FusedParams f) {
    using G = Geo<S>;
    constexpr int NW = G::NW, NWB = G::NWB, NB = G::NB, NT = G::NT, E = G::E, VS = G::VS, CPT = G::CPT;
    constexpr bool FAST = MODE == 1 || MODE == 2, FRAC = MODE == 2, QF = MODE == 4 || MODE == 5 || MODE == 6, CHI = MODE == 5,
                   P2Q = MODE == 6;
    extern __shared__ uint4 smem_raw[];
    uint32_t* vc = reinterpret_cast<uint32_t*>(smem_raw);                 // [NB bins][VS words], padded
    // integer paths over part of the histogram (!ALLB): running column counts of the group's
    // bins together, the window totals C of the group from one window-count pass per strip
    uint32_t* vcind = vc + NB * VS;                                         // [VS words]
    uint32_t* gbuf = vcind + VS;                                            // [NW warps][4][128 words] (general kw)
    // the group's window totals C per row parity, strip and window pair (packed): red32 for
    // the integer paths, gbuf for the quarter-layout FP32 paths (whose partials fill `red`)
    double* red = reinterpret_cast<double*>(gbuf + NW * 4 * kVcWords);      // [2 rows][NW warps][128]
    uint32_t* srep_s = reinterpret_cast<uint32_t*>(red + 2 * NW * kStrip);  // [NB]
    uint32_t* lrow = srep_s + NB;                                           // [2 rows][S strips][NB] row carries
    uint16_t* rowbins = reinterpret_cast<uint16_t*>(lrow + 2 * S * NB);     // [2 rows][S * 128] strip bins
    uint32_t* amask = reinterpret_cast<uint32_t*>(rowbins + 2 * kStrip * S);  // [8 lanes][8 words] anchor masks
    // integer path: [2 rows][128] earlier groups' sums (the FP64 path's part of `red`)
    double* accb = red + 2 * kStrip;
    // integer path: per row parity, strip and window pair, the packed sums over the warps
    // (shared atomics), I at [parity][strip][64] and C at 128 S + [parity][strip][64]
    uint32_t* red32 = reinterpret_cast<uint32_t*>(red);
    uint32_t* carea = (MODE == 4 || MODE == 5) ? gbuf : red32 + 128 * S;
    // fractional path, in 2^-40 fixed point (exact sums in any order): per row parity and
    // window the correction accumulated over the warps ([2][S][128] pairs of u32 shared
    // atomics on the low 24 bits and the rest of each warp's u64 value: no 64-bit CAS loop), and
    // per bin slab four 16-entry tables (one per flag nibble) of sums of r_k over 4 bins.
    // gbuf (16 KB) is unused by the integer paths; `red` holds red32 (S KB) and accb.
    uint64_t* acc64 = S == 8 ? reinterpret_cast<uint64_t*>(gbuf) : reinterpret_cast<uint64_t*>(red + 512);
    uint64_t* tab64 = S == 8 ? reinterpret_cast<uint64_t*>(red + 1024) : reinterpret_cast<uint64_t*>(gbuf);

    // Two variants are launched; the one that does not match the template prep exits.
    if (__ldg(f.prep) != static_cast<uint32_t>(MODE)) return;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sc = warp / NWB, wb = warp % NWB;            // the warp's strip in the CTA, bin slab
    const int strip = blockIdx.x * S + sc, band = blockIdx.y;
    const int g0 = f.group0;                               // slab-local first bin of the CTA
    const int nb_cta = min(NB, out.bins - g0);
    const int nwarps_live = (nb_cta + kB - 1) / kB;        // live bin slabs per strip
    const int kl0 = g0 + wb * kB;                          // warp's first slab-local bin
    const int xc = blockIdx.x * S * kStrip;                // CTA's first column
    const int xs = strip * kStrip;                         // warp's strip's first column
    const bool warp_live = wb < nwarps_live && strip < nstrips;
    const int k_live = min(kB, out.bins - kl0);
    const int xl = xs + 4 * lane;                          // lane's first strip column
    const int H = out.height, W = out.width;
    const int y0 = band * band_rows, y1 = min(H, y0 + band_rows);
    const int ystart = max(0, y0 - f.kh + 1);
    const int k0 = out.bin0 + kl0;                         // global bin of the warp's first plane
    const uint32_t kpat0 = pm.byte_mode ? 0x01010101u * static_cast<uint32_t>(k0) : 0u;
    const uint8_t* g8p = static_cast<const uint8_t*>(q.p0);
    auto raw_at = [&](int x, int y) -> uint64_t {
        if (SK == 1 || SK == 3) return static_cast<uint64_t>(__ldg(g8p + static_cast<int64_t>(y) * q.pitch + x));
        if (SK == 2) return static_cast<uint64_t>(__ldg(static_cast<const uint16_t*>(q.p0) + static_cast<int64_t>(y) * q.pitch + x));
        return pixel_raw(q, x, y);
    };
    auto bin_of = [&](uint64_t r) -> int {
        if (SK == 1 || SK == 3) return static_cast<int>((static_cast<uint32_t>(r) * static_cast<uint32_t>(q.nbins)) >> 8);
        if (SK == 2) return static_cast<int>(r);
        return bin_of_raw(r, q);
    };

    for (int i = tid; i < (NB + 1) * VS; i += NT) vc[i] = 0;
    if (FAST)
        for (int i = tid; i < 4 * 64 * S; i += NT) red32[i] = 0;  // row accumulators {I} [2][S][64], {C} [2][S][64]
    if (tid < NB) srep_s[tid] = (FAST && tid < nb_cta) ? __ldg(f.prep + 1 + g0 + tid) : 0u;
    if ((FAST || QF) && KWM == 0)
        for (int i = tid; i < 64; i += NT) {
            // anchor masks: u16 i of lane m's word j is valid iff 16m + 2j + i < kw
            const int n = f.kw - 16 * (i >> 3) - 2 * (i & 7);
            amask[i] = n >= 2 ? 0xFFFFFFFFu : (n == 1 ? 0xFFFFu : 0u);
        }
    if (FRAC) {
        // table n of slab wbi, index i: sum of r_k (2^-40 units) over the slab's bins 4 g + q(n)
        // with bit g of i set, q = {3, 1, 2, 0} for nibbles n = 0..3: the flag layout after the
        // cross-quarter combine below
        for (int i = tid; i < NWB * 64; i += NT) {
            const int wbi = i >> 6, n = (i >> 4) & 3, idx = i & 15;
            const int q = n == 0 ? 3 : (n == 1 ? 1 : (n == 2 ? 2 : 0));
            const int kb = g0 + wbi * kB + q, klim = g0 + nb_cta;
            uint64_t acc = 0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
                if (((idx >> g) & 1) && kb + 4 * g < klim)
                    acc += __double2ull_rn(__ldg(f.rfrac + kb + 4 * g) * 1099511627776.0);  // 2^40
            tab64[i] = acc;
        }
        for (int i = tid; i < 2 * kStrip * S; i += NT) acc64[i] = 0;
    }

    uint32_t V[4][kB];
    if (STORE && warp_live)
        vpart_init_ca<kB>(V, fc.C, fc.A, band, strip, gridDim.y, nstrips, Lb, Wp, kl0, xl);
    uint32_t* base_ptr = STORE ? out.data + static_cast<int64_t>(kl0) * out.plane_pitch + xl : nullptr;
    const bool lane_live = xl < out.row_pitch;
    const uint32_t store_mask = (lane_live && warp_live) ? (k_live >= 32 ? 0xFFFFFFFFu : (1u << max(k_live, 0)) - 1u) : 0u;
    const long long Sg = FAST ? f.S_group[g0 / kGroupBins] : 0;
    const double Sd = static_cast<double>(Sg) + (FRAC ? f.Sr_group[g0 / kGroupBins] : 0.0);  // sum of s_k
    // the warp's view of vc: ext columns [128 sc, 128 sc + 256) = padded words from 72 sc
    const uint32_t* vwarp = vc + wb * kB * VS + G::WOFF * sc;
    // general path: G(e - kw) as a word and a bit shift
    const int idx = kStrip + 4 * lane - f.kw;
    const int pw = idx >> 1, psh = (idx & 1) * 16;
    uint32_t* gb = gbuf + warp * 4 * kVcWords;
    // integer path: quarter qq of the warp takes bin 4g + qq; lane mq owns windows 16mq ..
    const int qq = lane >> 3, mq = lane & 7;
    const int ca0 = kStrip + 16 * mq - f.kw;  // extended column of vc(e - kw) for the lane's first window
    const int aw0 = ca0 >> 1, apsh = (ca0 & 1) * 16;
    const uint32_t* vq = vwarp + qq * VS;  // the quarter's bin row for g = 0
    const uint32_t* pb = vq + vcw(64 + 8 * mq);

    // staging: thread tid owns extended columns tid + c NT (c < CPT, col < E); their raw
    // pixels are prefetched one row ahead (32-bit raw values for the 8/16-bit sources; the
    // generic source with several columns per thread keeps the in-row loads)
    // (not for the slab variants of 4- and 8-strip CTAs: with the indicator row their
    // prefetch registers spill, which turns every prefetch into a stall; measured on the
    // 32 / 16-bin slabs of C3: 0.816 -> 0.770 / 0.554 -> 0.536 ms, tools/slab_time.py)
    constexpr bool WIDE = SK == 3;  // below
    constexpr bool PREFETCH = !WIDE && (CPT == 1 || (SK != 0 && (ALLB || S < 4)));
    using RawT = std::conditional_t<CPT == 1 || SK == 0, uint64_t, uint32_t>;
    int xt[CPT], vcol_w[CPT];
    bool xt_live[CPT];
    uint32_t vinc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int col = tid + c * NT;
        xt[c] = xc - kStrip + col;
        xt_live[c] = col < E && xt[c] >= 0 && xt[c] < W;
        vcol_w[c] = vcw(col >> 1);  // the column's (padded) vc word
        vinc[c] = 1u << (16 * (col & 1));
    }
    // row carries: thread tid < S NB loads those of bin tid % NB of strip tid / NB
    const int lt_strip = blockIdx.x * S + tid / NB;
    const uint16_t* lt_cta = (STORE && fc.Lt && tid < S * NB && lt_strip > 0 && lt_strip < nstrips &&
                              g0 + tid % NB < Lb)
                                 ? fc.Lt + static_cast<int64_t>(lt_strip) * H * Lb + g0 + tid % NB
                                 : nullptr;
    // raw pixel values of the staging column, quantised one row after the load
    RawT rn[CPT], ro[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        rn[c] = (PREFETCH && xt_live[c]) ? static_cast<RawT>(raw_at(xt[c], y0)) : 0;
        ro[c] = 0;
    }
    // WIDE (SK 3: 8-bit gray, 4-byte aligned rows; 4- and 8-strip CTAs): thread tid stages
    // the 4-column words tid + w NT of the extended row instead — one 32-bit load per word
    // and row for the entering and one for the leaving pixels, one 8-byte store of the
    // strip bins — a third of the per-column staging instructions, which weigh 4x more per
    // output byte at 32 bins than at 128
    constexpr int EW = E / 4, WPT = WIDE ? (EW + NT - 1) / NT : 1;
    bool xw_live[WPT];
    uint32_t rnw[WPT], row_[WPT];
#pragma unroll
    for (int w = 0; w < WPT; ++w) {
        const int wi = tid + w * NT, xw = xc - kStrip + 4 * wi;
        xw_live[w] = WIDE && wi < EW && xw >= 0 && xw < W;
        rnw[w] = xw_live[w] ? __ldg(reinterpret_cast<const uint32_t*>(g8p + static_cast<int64_t>(y0) * q.pitch + xw)) : 0u;
        row_[w] = 0;
    }
    bool have_o = false;  // y0 - kh < ystart: nothing to remove on the first row
    uint32_t lpre = lt_cta ? static_cast<uint32_t>(__ldg(lt_cta + static_cast<int64_t>(y0) * Lb)) : 0u;
    __syncthreads();  // vc zeroed

    // (narrow bin groups only: with 128 bins the table loads take as many rounds as the
    // pre-roll, and the branch alone costs the headline variant ~1.5%)
    if (NB < kGroupBins && fc.S && band > 0 && f.kh > 1) {
        // vc over rows [ystart, y0) from the carry tables (carries.cu): rows above y0 minus
        // rows above the band holding ystart, plus that band's suffix from ystart
        // (u16 pairs, every true count >= 0 and < 2^16, so no borrow crosses a half)
        const uint32_t* C32 = reinterpret_cast<const uint32_t*>(fc.C);
        const uint32_t* S32 = reinterpret_cast<const uint32_t*>(fc.S);
        const int64_t plane = static_cast<int64_t>(Lb) * Wp / 2;  // words per band
        const int r = y0 - f.kh + 1, ib = r > 0 ? r / band_rows : -1;
        constexpr int U = 8;  // loads in flight per thread
        const int n = nb_cta * G::VW;
        for (int i0 = tid; i0 < n; i0 += U * NT) {
            uint32_t pj[U], sf[U], pi[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NT;
                const int k = i / G::VW, w = i % G::VW;  // bin, extended-column word (columns 2w, 2w + 1)
                const int x = xc - kStrip + 2 * w;
                const bool live = i < n && x >= 0 && x < Wp;
                const int64_t off = ((static_cast<int64_t>(g0 + k) * Wp) + x) >> 1;
                pj[u] = live ? __ldg(C32 + (band - 1) * plane + off) : 0u;
                sf[u] = (live && ib >= 0) ? __ldg(S32 + ib * plane + off) : 0u;
                pi[u] = (live && ib >= 0 && ib + 1 < band) ? __ldg(C32 + ib * plane + off) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NT;
                if (i < n) vc[(i / G::VW) * VS + vcw(i % G::VW)] = ib < 0 ? pj[u] : (ib + 1 == band ? sf[u] : sf[u] + pj[u] - pi[u]);
            }
        }
    } else {
        // No tables (tensor not stored, or 128 bins): pre-roll rows [ystart, y0) only feed
        // vc, and nothing leaves the window there: one barrier-free pass with several loads
        // in flight (a per-row loop would pay the full DRAM latency on every row).
#pragma unroll
        for (int c = 0; c < CPT; ++c)
            if (xt_live[c]) {
                const int nb_lo = out.bin0 + g0;
                uint32_t* vcol = vc + vcol_w[c];
                for (int y = ystart; y < y0; y += 8) {
                    uint64_t r[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) r[i] = y + i < y0 ? raw_at(xt[c], y + i) : 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int bn = bin_of(r[i]) - nb_lo;
                        if (y + i < y0 && static_cast<unsigned>(bn) < static_cast<unsigned>(nb_cta))
                            atomicAdd(vcol + bn * VS, vinc[c]);
                    }
                }
            }
    }
    constexpr bool IND = (FAST || CHI) && !ALLB;  // the group indicator row is kept
    if (IND) {  // band start: the indicator's column counts are the sum of the bins' (u16 pairs <= kh)
        __syncthreads();
        for (int i = tid; i < VS; i += NT) {
            uint32_t acc = 0;
            for (int k = 0; k < nb_cta; ++k) acc += vc[k * VS + i];
            vcind[i] = acc;
        }
    }

    // row yy's partials are in `red` (and must be combined) iff it is a match row
    auto pending_row = [&](int yy) { return yy >= y0 && yy >= f.kh - 1; };
    auto pending = pending_row;
    // Cross-warp combine of row yy: thread t < 128 S finishes the window ending at CTA
    // column t.  Integer path with a finished map (ALLB): L = alpha + beta I (one FMA).
    const bool intersect = f.metric == SPCT_METRIC_INTERSECTION;
    const double lin_b = f.invT;
    const double lin_a = intersect ? 0.0 : 1.0 - (static_cast<double>(static_cast<long long>(f.kw) * f.kh) + Sd) * f.invT * 0.5;
    auto write_map = [&](int u, int v, double L) {
        // spread_valid's border replication (likelihood.cpp:44-58)
        const int x = u + (f.kw - 1) / 2, yc = v + (f.kh - 1) / 2;
        if (u > 0 && u < f.nu - 1 && v > 0 && v < f.nv - 1) {
            f.map[static_cast<int64_t>(yc) * f.W + x] = L;
            return;
        }
        const int xa = u == 0 ? 0 : x, xb = u == f.nu - 1 ? f.W - 1 : x;
        const int ya = v == 0 ? 0 : yc, yb = v == f.nv - 1 ? f.H - 1 : yc;
        for (int yy = ya; yy <= yb; ++yy)
            for (int xx = xa; xx <= xb; ++xx) f.map[static_cast<int64_t>(yy) * f.W + xx] = L;
    };
    // accumulate (bin groups after the first): the earlier groups' partial sum of the
    // window combined next, loaded one row ahead so the combine never waits on DRAM
    // (S == 1, the only geometry with several groups: thread t < 128 owns window t)
    // (cp.async into a per-thread shared slot: no register is held across the row)
    auto load_acc = [&](int yy) {
        if (FAST && S == 1 && f.accumulate && tid < kStrip && pending_row(yy)) {
            const int e = xc + tid, u = e - f.kw + 1;
            if (u >= 0 && e < W) {
                const double* src = f.partial + static_cast<int64_t>(yy - f.kh + 1) * f.nu + u;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n\tcp.async.commit_group;" ::"r"(
                                 static_cast<uint32_t>(__cvta_generic_to_shared(accb + (yy & 1) * kStrip + tid))),
                             "l"(src)
                             : "memory");
            }
        }
    };
    auto add_acc = [&](int yy, int u, int v, double term) {
        if (!f.accumulate) return term;
        if (FAST && S == 1) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            return __dadd_rn(accb[(yy & 1) * kStrip + tid], term);
        }
        return __dadd_rn(f.partial[static_cast<int64_t>(v) * f.nu + u], term);
    };
    auto combine_one = [&](int yy, int t) {
        const int e = xc + t;
        const int u = e - f.kw + 1, v = yy - f.kh + 1;
        if (FAST) {
            // the warps' packed window-pair sums, accumulated in shared memory; every
            // sum stays below 2^16 (at most kw * kh).  Read, then clear for row yy + 2.
            uint32_t* ai = red32 + (yy & 1) * 64 * S + (t >> 1);
            const uint32_t xi = *ai;
            const uint32_t xcn = ALLB ? 0u : carea[(yy & 1) * 64 * S + (t >> 1)];  // rewritten every row
            __syncwarp();
            if (!(t & 1)) *ai = 0;
            if (u < 0 || e >= W) return;
            const uint32_t I = (xi >> (16 * (t & 1))) & 0xFFFFu;
            // sum_k min(c_k, s_k): exact integers, plus the fractional correction (2^-40 fixed
            // point: within 2^-41 per bin of sum r_k, independent of the summation order)
            double Id = static_cast<double>(I);
            if (FRAC) {
                uint64_t* a64 = acc64 + (yy & 1) * kStrip * S + t;
                const uint2 pr = *reinterpret_cast<const uint2*>(a64);
                *a64 = 0;  // for row yy + 2
                const uint64_t corr = (static_cast<uint64_t>(pr.y) << 24) + pr.x;
                Id += static_cast<double>(corr) * (1.0 / 1099511627776.0);
            }
            if (ALLB && f.map) {
                const double L = fma(lin_b, Id, lin_a);
                write_map(u, v, fmin(fmax(L, 0.0), 1.0));
                return;
            }
            const long long C = ALLB ? static_cast<long long>(f.kw) * f.kh : (xcn >> (16 * (t & 1))) & 0xFFFFu;
            const double term = add_acc(yy, u, v, intersect ? Id * f.invT
                                                        : (FRAC ? (static_cast<double>(C) + Sd - 2.0 * Id) * f.invT
                                                                : static_cast<double>(C + Sg - 2 * static_cast<long long>(I)) * f.invT));
            if (f.map) write_map(u, v, finalize_L(term, f));  // the last group finishes the map
            else f.partial[static_cast<int64_t>(v) * f.nu + u] = term;
        } else {
            if (u < 0 || e >= W) return;
            const double* rb = red + (yy & 1) * (NW * kStrip) + (t / kStrip) * NWB * kStrip + (t % kStrip);
            double term = 0.0;
#pragma unroll
            for (int w = 0; w < NWB; ++w)
                if (w < nwarps_live) term = __dadd_rn(term, rb[w * kStrip]);
            if (CHI) {  // + C / T, C the window's count over the group's bins
                const uint32_t cn = ALLB ? 0u : carea[(yy & 1) * 64 * S + (t >> 1)];
                const double C = ALLB ? static_cast<double>(f.kw) * f.kh : static_cast<double>((cn >> (16 * (t & 1))) & 0xFFFFu);
                term = __dadd_rn(term, C * f.invT);
            }
            term = add_acc(yy, u, v, term);
            if (f.map) write_map(u, v, finalize_L(term, f));
            else f.partial[static_cast<int64_t>(v) * f.nu + u] = term;
        }
    };
    // exact integer path into a finished map with several strips per CTA: thread t finishes
    // the window pair (2 t, 2 t + 1), whose packed sums share one word: one read and clear
    // (no other thread touches the word) and one 16-byte store for an interior pair
    constexpr bool PAIRS = MODE == 1 && ALLB && S >= 2;
    const bool map_even = PAIRS && f.map && (reinterpret_cast<uintptr_t>(f.map) & 15) == 0 && (f.W & 1) == 0;
    auto combine_pair = [&](int yy, int t2) {
        uint32_t* ai = red32 + (yy & 1) * 64 * S + t2;
        const uint32_t xi = *ai;
        *ai = 0;  // for row yy + 2
        const int e = xc + 2 * t2;
        const int u = e - f.kw + 1, v = yy - f.kh + 1;
        const double L0 = fmin(fmax(fma(lin_b, static_cast<double>(xi & 0xFFFFu), lin_a), 0.0), 1.0);
        const double L1 = fmin(fmax(fma(lin_b, static_cast<double>(xi >> 16), lin_a), 0.0), 1.0);
        const int x = u + (f.kw - 1) / 2, yc = v + (f.kh - 1) / 2;
        if (map_even && u > 0 && u + 1 < f.nu - 1 && v > 0 && v < f.nv - 1 && !(x & 1)) {
            *reinterpret_cast<double2*>(f.map + static_cast<int64_t>(yc) * f.W + x) = make_double2(L0, L1);
            return;
        }
        if (u >= 0 && e < W) write_map(u, v, L0);
        if (u + 1 >= 0 && e + 1 < W) write_map(u + 1, v, L1);
    };
    auto combine = [&](int yy) {
        if (PAIRS && f.map) {
#pragma unroll
            for (int t2 = tid; t2 < 64 * S; t2 += NT) combine_pair(yy, t2);
            return;
        }
#pragma unroll
        for (int t = tid; t < kStrip * S; t += NT) combine_one(yy, t);
    };


    // The strip's window totals over the group's bins (paths that need C and do not hold
    // the whole histogram): one window-count pass over the indicator row per strip and row
    // (every quarter of the strip's first warp computes it; quarter 0 stores the 128)
    auto ind_pass = [&](int y) {
        if (IND && wb == 0) {
            const uint32_t* vwi = vcind + G::WOFF * sc;
            uint32_t cw[8];
            int coff;
            window_counts_q<KWM>(vwi + vcw(64 + 8 * mq), vwi, mq, aw0, apsh, amask, cw, coff);
            if (qq == 0) {
                uint32_t* cr = carea + (y & 1) * 64 * S + sc * 64 + 8 * mq;
#pragma unroll
                for (int j = 0; j < 8; ++j) cr[j] = cw[j] + static_cast<uint32_t>(coff) * 0x10001u;
            }
        }
    };

    for (int y = y0; y < y1; ++y) {
        __syncthreads();  // A: previous row's vc / staging reads are done, its partials written
        // row y - 1's partials were written before A; its buffer is rewritten only after
        // the next B.  Some warps combine while the others start staging.
        if (pending(y - 1)) combine(y - 1);
        load_acc(y);
        {   // stage row y: vertical running histogram (add row y, remove row y - kh),
            // the strips' bins and row carries for the sweep, then prefetch row y + 1
            const bool old_row = y - f.kh >= ystart;
            if (WIDE) {
#pragma unroll
                for (int w = 0; w < WPT; ++w) {
                    const int wi = tid + w * NT;
                    const int xw = xc - kStrip + 4 * wi;
                    uint32_t* vw = vc + vcw(2 * wi);  // columns 4 wi, +1 (word 2 wi) and +2, +3 (the next)
                    uint32_t pk[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};  // strip bins, 0xFFFF past the image
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (!xw_live[w] || xw + j >= W) break;
                        const uint32_t inc = 1u << (16 * (j & 1));
                        const int pn = static_cast<int>((((rnw[w] >> (8 * j)) & 0xFFu) * static_cast<uint32_t>(q.nbins)) >> 8);
                        const int bn = pn - out.bin0 - g0;
                        const bool in_n = static_cast<unsigned>(bn) < static_cast<unsigned>(nb_cta);
                        if (in_n) atomicAdd(vw + bn * VS + (j >> 1), inc);
                        bool in_o = false;
                        if (have_o) {
                            const int po = static_cast<int>((((row_[w] >> (8 * j)) & 0xFFu) * static_cast<uint32_t>(q.nbins)) >> 8);
                            const int bo = po - out.bin0 - g0;
                            in_o = static_cast<unsigned>(bo) < static_cast<unsigned>(nb_cta);
                            if (in_o) atomicSub(vw + bo * VS + (j >> 1), inc);
                        }
                        if (IND && in_n != in_o) atomicAdd(vcind + vcw(2 * wi) + (j >> 1), in_n ? inc : 0u - inc);
                        pk[j >> 1] = (pk[j >> 1] & ~(0xFFFFu << (16 * (j & 1)))) | (static_cast<uint32_t>(pn) << (16 * (j & 1)));
                    }
                    if (4 * wi >= kStrip && wi < EW)
                        *reinterpret_cast<uint2*>(rowbins + (y & 1) * kStrip * S + 4 * wi - kStrip) = make_uint2(pk[0], pk[1]);
                }
            }
#pragma unroll
            for (int c = 0; c < (WIDE ? 0 : CPT); ++c) {
                const uint64_t rnc = PREFETCH ? rn[c] : (xt_live[c] ? raw_at(xt[c], y) : 0);
                const uint64_t roc = PREFETCH ? ro[c] : ((xt_live[c] && old_row) ? raw_at(xt[c], y - f.kh) : 0);
                const bool ho = PREFETCH ? have_o : old_row;
                const int pn = xt_live[c] ? bin_of(rnc) : 0xFFFF;
                const int po = (xt_live[c] && ho) ? bin_of(roc) : -1;
                if (xt_live[c]) {
                    const int bn = pn - out.bin0 - g0;
                    const bool in_n = static_cast<unsigned>(bn) < static_cast<unsigned>(nb_cta);
                    if (in_n) atomicAdd(&vc[bn * VS + vcol_w[c]], vinc[c]);
                    const int bo = po - out.bin0 - g0;
                    const bool in_o = po >= 0 && static_cast<unsigned>(bo) < static_cast<unsigned>(nb_cta);
                    if (in_o) atomicSub(&vc[bo * VS + vcol_w[c]], vinc[c]);
                    if (IND && in_n != in_o) atomicAdd(&vcind[vcol_w[c]], in_n ? vinc[c] : 0u - vinc[c]);
                }
                const int col = tid + c * NT;
                if (col >= kStrip && col < E) rowbins[(y & 1) * kStrip * S + col - kStrip] = static_cast<uint16_t>(pn);
            }
            if (tid < S * NB) lrow[(y & 1) * S * NB + tid] = lpre;
            if (y + 1 < y1) {
                if (WIDE) {
                    const int yo = y + 1 - f.kh;
                    have_o = yo >= ystart;
#pragma unroll
                    for (int w = 0; w < WPT; ++w)
                        if (xw_live[w]) {
                            const uint8_t* cp = g8p + xc - kStrip + 4 * (tid + w * NT);
                            rnw[w] = __ldg(reinterpret_cast<const uint32_t*>(cp + static_cast<int64_t>(y + 1) * q.pitch));
                            if (have_o) row_[w] = __ldg(reinterpret_cast<const uint32_t*>(cp + static_cast<int64_t>(yo) * q.pitch));
                        }
                } else if (PREFETCH) {
                    const int yo = y + 1 - f.kh;
                    have_o = yo >= ystart;
#pragma unroll
                    for (int c = 0; c < CPT; ++c)
                        if (xt_live[c]) {
                            rn[c] = static_cast<RawT>(raw_at(xt[c], y + 1));
                            if (have_o) ro[c] = static_cast<RawT>(raw_at(xt[c], yo));
                        }
                }
                if (lt_cta) lpre = __ldg(lt_cta + static_cast<int64_t>(y + 1) * Lb);
            }
        }
        __syncthreads();  // B: vc holds rows (y - kh, y]; staging rows ready
        const bool match_row = y >= f.kh - 1;
        if (!warp_live || (!STORE && !match_row)) continue;

        uint32_t t4[4] = {0, 0, 0, 0};
        if (STORE) {
            const uint2 rb2 = *reinterpret_cast<const uint2*>(rowbins + (y & 1) * kStrip * S + sc * kStrip + 4 * lane);
            uint32_t bins4 = 0;
            if (pm.byte_mode) {
                bins4 = __byte_perm(rb2.x, rb2.y, 0x6420);
            } else {
                const uint32_t b4[4] = {rb2.x & 0xFFFFu, rb2.x >> 16, rb2.y & 0xFFFFu, rb2.y >> 16};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t r = b4[j] - static_cast<uint32_t>(k0);
                    bins4 |= (r < static_cast<uint32_t>(kB) ? r : 0xFFu) << (8 * j);
                }
            }
            onehot_shifts(bins4 ^ kpat0, t4);
        }
        const uint4* lr = reinterpret_cast<const uint4*>(lrow + (y & 1) * S * NB + sc * NB + wb * kB);
        uint32_t* prow = STORE ? base_ptr + static_cast<int64_t>(y) * out.row_pitch : nullptr;

        uint32_t Iw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int Ioff = 0;  // per-lane offset summed over the lane's bins (integer path)
        // fractional path: flag of c_k > floor(s_k) for group g at bit 12 + g of each half
        uint32_t Pf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pall = 0;
        // MODE 4: the lane's 16 windows' FP32 sums over its four bins
        [[maybe_unused]] float qf[16];
        [[maybe_unused]] int qi[16];  // MODE 6: the exact integer part of the p = 2 terms
        if (QF)
#pragma unroll
            for (int i = 0; i < 16; ++i) qf[i] = 0.0f;
        if (P2Q)
#pragma unroll
            for (int i = 0; i < 16; ++i) qi[i] = 0;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int g = 0; g < kB / 4; ++g) {
            if (STORE)
                vpart_group_q<kB>(V, g, t4, lr[g], prow + static_cast<int64_t>(4 * g) * out.plane_pitch, out.plane_pitch,
                                  store_mask);
            if (QF && match_row) {
                uint32_t w[8];
                int off;
                const int go = 4 * g * VS;
                window_counts_q<KWM>(pb + go, vq + go, mq, aw0, apsh, amask, w, off);
                const int kq = kl0 + 4 * g + qq;  // the quarter's bin (slab-local)
                const float4 cst = kq < out.bins ? __ldg(f.c3 + kq) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                // c = half + off exactly in FP32: 2^23 + half by bit pattern, plus off - 2^23
                const float cfo = static_cast<float>(off) - 8388608.0f;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float c0 = __int_as_float(0x4B000000u | (w[j] & 0xFFFFu)) + cfo;
                    const float c1 = __int_as_float(0x4B000000u | (w[j] >> 16)) + cfo;
                    if (P2Q) {  // (c - s)^2 as MODE 3: c (32 c - X) exact in int32, c Y in FP32
                        const int i0 = static_cast<int>(w[j] & 0xFFFFu) + off, i1 = static_cast<int>(w[j] >> 16) + off;
                        qi[2 * j] += i0 * (32 * i0 - __float_as_int(cst.x));
                        qi[2 * j + 1] += i1 * (32 * i1 - __float_as_int(cst.x));
                        qf[2 * j] = fmaf(c0, cst.y, qf[2 * j]);
                        qf[2 * j + 1] = fmaf(c1, cst.y, qf[2 * j + 1]);
                    } else if (CHI) {  // c s / (c + s); c = s = 0 gives 0 (the reference skips q + t = 0)
                        qf[2 * j] = fmaf(c0 * cst.w, rcp_approx(c0 + cst.w + 1e-30f), qf[2 * j]);
                        qf[2 * j + 1] = fmaf(c1 * cst.w, rcp_approx(c1 + cst.w + 1e-30f), qf[2 * j + 1]);
                    } else {    // sqrt(c) sqrt(t / T)
                        qf[2 * j] = fmaf(sqrt_approx(c0), cst.z, qf[2 * j]);
                        qf[2 * j + 1] = fmaf(sqrt_approx(c1), cst.z, qf[2 * j + 1]);
                    }
                }
            }
            if (FAST && match_row) {
                uint32_t w[8];
                int off;
                const int go = 4 * g * VS;
                window_counts_q<KWM>(pb + go, vq + go, mq, aw0, apsh, amask, w, off);
                const int sk = static_cast<int>(srep_s[wb * kB + 4 * g + qq] & 0xFFFFu);
                // min(w + off, s_k) = min(w, s_k - off) + off.  A negative threshold (off > s_k:
                // e.g. a window inside one bin against a template with < 16 pixels of it) has
                // min = s_k - off for every w >= 0: it goes to the offset and the packed min
                // runs on 0, so every half stays a non-negative u16 (exact linear encoding).
                // 0 <= thr <= s_k + 8160 < 2^16.
                const int ti = sk - off;
                const uint32_t thr = static_cast<uint32_t>(max(ti, 0)) * 0x10001u;
                constexpr uint32_t kFlag = 0x10001u << 12;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t mn = min_u16x2(w[j], thr);
                    Iw[j] += mn;
                    // d = w - min = max(c - floor(s), 0) <= kw kh <= 4096 per half: bit 12 + g
                    // of d + 2^(12+g) - 1 is set iff d >= 1 (no carry across the halves)
                    if (FRAC) Pf[j] |= (w[j] - mn + (kFlag << g) - 0x10001u) & (kFlag << g);
                }
                Ioff += off + min(ti, 0);
                if (FRAC) pall |= ti < 0 ? (kFlag << g) : 0u;  // c > floor(s) in every window

            }
        }
        if constexpr (!FAST && !QF) if (match_row) {
            // FP64 path (MODE 0) / integer-FP32 terms (MODE 3): the window terms in a rolled loop
            // over the bin groups, one loop per metric (a per-row switch) so the running loop
            // stays small
            auto rows = [&](auto fk_tag) {
                constexpr int FK = decltype(fk_tag)::value;
                [[maybe_unused]] const double invT = f.invT, pp = f.p;
                [[maybe_unused]] int ai[4] = {0, 0, 0, 0};  // MODE 3
                [[maybe_unused]] float af[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                [[maybe_unused]] uint32_t cw[2] = {0u, 0u};  // MODE 3, chi-square: packed window counts
#pragma unroll 1
                for (int g = 0; g < kB / 4; ++g) {
                    uint32_t aw[4][2], bw[4][2];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        window_prefix<KWM == 0>(vwarp + (4 * g + i) * VS, gb + i * kVcWords, lane, aw[i][0],
                                                aw[i][1], bw[i][0], bw[i][1]);
                    if (KWM == 0) __syncwarp();
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int k = 4 * g + i;
                        uint32_t c0, c1;
                        if (KWM == 64) {
                            // G(e - 64): the partner lane^16's halo half (lanes < 16) or strip half (>= 16)
                            const uint32_t r0 = __shfl_xor_sync(0xffffffffu, lane >= 16 ? aw[i][0] : bw[i][0], 16);
                            const uint32_t r1 = __shfl_xor_sync(0xffffffffu, lane >= 16 ? aw[i][1] : bw[i][1], 16);
                            c0 = bw[i][0] - r0;
                            c1 = bw[i][1] - r1;
                        } else if (KWM == 128) {
                            c0 = bw[i][0] - aw[i][0];  // G(e - 128) is the lane's own halo half
                            c1 = bw[i][1] - aw[i][1];
                        } else {
                            window_diff(gb + i * kVcWords, pw, psh, bw[i][0], bw[i][1], c0, c1);
                        }
                        if constexpr (MODE == 3) {
                            if (k < k_live) {
                                const float4 cst = __ldg(f.c3 + kl0 + k);
                                if (FK == 5) {
                                    cw[0] += c0;
                                    cw[1] += c1;
                                }
                                if (FK != 5 || cst.w > 0.0f) {  // chi-square: bins with s = 0 add 0 to Y
                                    f32_term<FK>(c0 & 0xFFFFu, cst, ai[0], af[0]);
                                    f32_term<FK>(c0 >> 16, cst, ai[1], af[1]);
                                    f32_term<FK>(c1 & 0xFFFFu, cst, ai[2], af[2]);
                                    f32_term<FK>(c1 >> 16, cst, ai[3], af[3]);
                                }
                            }
                        } else if (k < k_live) {
                            const double t = __ldg(f.tmpl + k0 + k);
                            acc[0] = __dadd_rn(acc[0], fp_term<FK>(c0 & 0xFFFFu, t, invT, pp));
                            acc[1] = __dadd_rn(acc[1], fp_term<FK>(c0 >> 16, t, invT, pp));
                            acc[2] = __dadd_rn(acc[2], fp_term<FK>(c1 & 0xFFFFu, t, invT, pp));
                            acc[3] = __dadd_rn(acc[3], fp_term<FK>(c1 >> 16, t, invT, pp));
                        }
                    }
                    if (KWM == 0) __syncwarp();
                }
                if constexpr (MODE == 3) {
                    // the warp's partial term per window, in the units of the FP64 path
                    const double2 sc = f.c3slab[kl0 / kB];  // {sum s^2, sum s} over the warp's bins
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (FK == 1) {
                            acc[j] = (static_cast<double>(ai[j]) * (1.0 / 32.0) - 2.0 * static_cast<double>(af[j]) + sc.x) *
                                     invT * invT;
                        } else if (FK == 4) {
                            acc[j] = static_cast<double>(af[j]);
                        } else {
                            const uint32_t cj = (cw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
                            acc[j] = (static_cast<double>(cj) + sc.y - 4.0 * static_cast<double>(af[j])) * invT;
                        }
                    }
                }
            };
            if constexpr (MODE == 3) {
                switch (f.fp_kind) {
                    case 1: rows(std::integral_constant<int, 1>{}); break;
                    case 4: rows(std::integral_constant<int, 4>{}); break;
                    default: rows(std::integral_constant<int, 5>{}); break;
                }
            } else switch (f.fp_kind) {
                case 0: rows(std::integral_constant<int, 0>{}); break;
                case 1: rows(std::integral_constant<int, 1>{}); break;
                case 2: rows(std::integral_constant<int, 2>{}); break;
                case 3: rows(std::integral_constant<int, 3>{}); break;
                case 4: rows(std::integral_constant<int, 4>{}); break;
                default: rows(std::integral_constant<int, 5>{}); break;
            }
        }
        if (match_row) {
            if (FAST) {
                // the quarters hold the same 16 windows per lane for different bins
#pragma unroll
                for (int j = 0; j < 8; ++j) Iw[j] += static_cast<uint32_t>(Ioff) * 0x10001u;
                quarter_reduce(Iw, qq);
                const int jb = 4 * (qq >> 1) + 2 * (qq & 1);
                if (FRAC) {
                    // combine the four quarters' flags of the lane's windows (the words jb, jb + 1
                    // of quarter_reduce): per half, quarter 0 / 2 / 1 / 3 at bits 12-15 / 8-11 /
                    // 4-7 / 0-3, then one table lookup per nibble and window
                    const bool hi2 = qq & 2, hi1 = qq & 1;
                    uint32_t v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t a = Pf[j] | pall, b = Pf[j + 4] | pall;
                        const uint32_t r = __shfl_xor_sync(0xffffffffu, hi2 ? a : b, 16);
                        v[j] = hi2 ? (r | (b >> 4)) : (a | (r >> 4));
                    }
                    uint32_t u2[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const uint32_t r = __shfl_xor_sync(0xffffffffu, hi1 ? v[j] : v[j + 2], 8);
                        u2[j] = hi1 ? (r | (v[j + 2] >> 8)) : (v[j] | (r >> 8));
                    }
                    const uint64_t* tb = tab64 + wb * 64;
                    uint64_t* a64 = acc64 + ((y & 1) * S + sc) * kStrip + 16 * mq + 2 * jb;
#pragma unroll
                    for (int h = 0; h < 4; ++h) {  // window 16 mq + 2 jb + h: half h & 1 of word h >> 1
                        const uint32_t x = u2[h >> 1] >> (16 * (h & 1));
                        const uint64_t v = tb[x & 15u] + tb[16 + ((x >> 4) & 15u)] + tb[32 + ((x >> 8) & 15u)] +
                                           tb[48 + ((x >> 12) & 15u)];
                        // v < 16 * 2^40: the low 24 bits and the high 20 summed over <= 8 warps fit u32
                        uint32_t* a32 = reinterpret_cast<uint32_t*>(a64 + h);
                        atomicAdd(a32, static_cast<uint32_t>(v) & 0xFFFFFFu);
                        atomicAdd(a32 + 1, static_cast<uint32_t>(v >> 24));
                    }
                }
                uint32_t* rw = red32 + (y & 1) * 64 * S + sc * 64 + 8 * mq + jb;
                if (NWB == 1) {  // one warp per strip: the row's sums are final
                    rw[0] = Iw[0];
                    rw[1] = Iw[1];
                } else {
                    atomicAdd(rw, Iw[0]);
                    atomicAdd(rw + 1, Iw[1]);
                }
                ind_pass(y);
            } else if (QF) {
                ind_pass(y);
                // the four quarters' sums of the same windows (reduce-scatter as quarter_reduce:
                // the lane keeps windows 16 mq + 8 hi2 + 4 hi1 + 0..3), then the warp's partial
                const bool hi2 = qq & 2, hi1 = qq & 1;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float snd = hi2 ? qf[i] : qf[i + 8], kp = hi2 ? qf[i + 8] : qf[i];
                    qf[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
                    if (P2Q) {
                        const int sn = hi2 ? qi[i] : qi[i + 8], kq = hi2 ? qi[i + 8] : qi[i];
                        qi[i] = kq + __shfl_xor_sync(0xffffffffu, sn, 16);
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float snd = hi1 ? qf[i] : qf[i + 4], kp = hi1 ? qf[i + 4] : qf[i];
                    qf[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
                    if (P2Q) {
                        const int sn = hi1 ? qi[i] : qi[i + 4], kq = hi1 ? qi[i + 4] : qi[i];
                        qi[i] = kq + __shfl_xor_sync(0xffffffffu, sn, 8);
                    }
                }
                double* rb = red + (y & 1) * (NW * kStrip) + warp * kStrip + 16 * mq + 8 * (qq >> 1) + 4 * (qq & 1);
                if (P2Q) {  // the warp's (sum c^2 - 2 sum c s + sum s^2) / T^2 (MODE 3's units)
                    const double s2 = f.c3slab[kl0 / kB].x;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        rb[i] = (static_cast<double>(qi[i]) * (1.0 / 32.0) - 2.0 * static_cast<double>(qf[i]) + s2) * f.invT *
                                f.invT;
                } else if (CHI) {  // the warp's (S_w - 4 Y_w) / T, S_w = sum of s_k over its bins
                    const double sw = f.c3slab[kl0 / kB].y;
#pragma unroll
                    for (int i = 0; i < 4; ++i) rb[i] = (sw - 4.0 * static_cast<double>(qf[i])) * f.invT;
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) rb[i] = static_cast<double>(qf[i]);
                }
            } else {
                double* rb = red + (y & 1) * (NW * kStrip) + warp * kStrip;
                rb[4 * lane + 0] = acc[0];
                rb[4 * lane + 1] = acc[1];
                rb[4 * lane + 2] = acc[2];
                rb[4 * lane + 3] = acc[3];
            }
        }
    }
    __syncthreads();
    if (y1 > y0 && pending(y1 - 1)) combine(y1 - 1);
}

constexpr size_t kSmemBytes = smem_bytes_s<1>();


template <int KWM, bool ALLB, int SK, int S>
void launch_variants(bool frac, int path, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm,
                     const spct_ih& out, const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f) {
    constexpr int NT = Geo<S>::NT;
    constexpr size_t SM = smem_bytes_s<S>();
    // the exact integer (template-crop) variant and, for the other templates, the
    // fractional variant (p = 1 / intersection, kw kh <= 4096) or the FP64 one: the variant
    // not selected by the device-side template prep exits on entry
#define SPCT_GO(ST, MD, AB)                                                                                      \
    {                                                                                                            \
        ensure_smem(sweep_match_kernel<ST, MD, KWM, AB, SK, S>, SM);                                             \
        sweep_match_kernel<ST, MD, KWM, AB, SK, S>                                                               \
            <<<grid, NT, SM, s>>>(q, pm, out, bp.Lb, bp.Wp, bp.band_rows, bp.nstrips, fc, f);                    \
    }
    // (a metric without an integer path launches its one variant: FP32 terms or FP64)
    if (out.data) {
        if (path == 1) {
            SPCT_GO(true, 1, ALLB)
            if (frac) SPCT_GO(true, 2, ALLB) else SPCT_GO(true, 0, false)
        } else if (path == 3) {
            SPCT_GO(true, 3, false)
        } else if (path == 4) {
            SPCT_GO(true, 4, false)
        } else if (path == 5) {
            SPCT_GO(true, 5, false)
        } else if (path == 6) {
            SPCT_GO(true, 6, false)
        } else {
            SPCT_GO(true, 0, false)
        }
    } else {
        if (path == 1) {
            SPCT_GO(false, 1, ALLB)
            if (frac) SPCT_GO(false, 2, ALLB) else SPCT_GO(false, 0, false)
        } else if (path == 3) {
            SPCT_GO(false, 3, false)
        } else if (path == 4) {
            SPCT_GO(false, 4, false)
        } else if (path == 5) {
            SPCT_GO(false, 5, false)
        } else if (path == 6) {
            SPCT_GO(false, 6, false)
        } else {
            SPCT_GO(false, 0, false)
        }
    }
#undef SPCT_GO
}

template <int KWM, int S>
void launch_kw_impl(bool allb, int sk, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm,
                    const spct_ih& out, const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f) {
#define SPCT_SK(SKV)                                                                      \
    if (allb) launch_variants<KWM, true, SKV, S>(f.frac, f.path, grid, s, q, pm, out, bp, fc, f);   \
    else launch_variants<KWM, false, SKV, S>(f.frac, f.path, grid, s, q, pm, out, bp, fc, f);
    if (sk == 3) {
        if constexpr (S >= 4) {  // (2- and 1-strip CTAs: 0.97 -> 1.19 / 1.83 -> 1.93 ms measured, the
            SPCT_SK(3)               // per-thread atomics of four columns lengthen their row)
        } else {
            SPCT_SK(1)
        }
    } else if (sk == 1) {
        SPCT_SK(1)
    } else if (sk == 2) {
        SPCT_SK(2)
    } else {
        SPCT_SK(0)
    }
#undef SPCT_SK
}

}  // namespace spct_fused

namespace spct_fused {
// One translation unit per (window-width specialisation, strips per CTA), so the kernel
// variants compile in parallel: fused_kw{64,128,0}_s{1,2,4,8}.cu.
#define SPCT_FUSED_LAUNCHER(NAME)                                                                              \
    void NAME(bool allb, int sk, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm,        \
              const spct_ih& out, const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f);
SPCT_FUSED_LAUNCHER(launch_kw64_s1)
SPCT_FUSED_LAUNCHER(launch_kw64_s2)
SPCT_FUSED_LAUNCHER(launch_kw64_s4)
SPCT_FUSED_LAUNCHER(launch_kw64_s8)
SPCT_FUSED_LAUNCHER(launch_kw128_s1)
SPCT_FUSED_LAUNCHER(launch_kw128_s2)
SPCT_FUSED_LAUNCHER(launch_kw128_s4)
SPCT_FUSED_LAUNCHER(launch_kw128_s8)
SPCT_FUSED_LAUNCHER(launch_kw_any_s1)
SPCT_FUSED_LAUNCHER(launch_kw_any_s2)
SPCT_FUSED_LAUNCHER(launch_kw_any_s4)
SPCT_FUSED_LAUNCHER(launch_kw_any_s8)
#undef SPCT_FUSED_LAUNCHER
size_t smem_bytes();
// Strips per CTA of the fused sweep for a slab of `bins` bins (1, 2, 4 or 8): every CTA has
// 8 warps of 16 bins.
inline int fused_strips(int bins) { return bins > 64 ? 1 : (bins > 32 ? 2 : (bins > 16 ? 4 : 8)); }
}  // namespace spct_fused
