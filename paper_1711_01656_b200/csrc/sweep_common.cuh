// The per-row integral-histogram update shared by the build sweep and the fused
// build+match sweep.
//
// A warp owns a 128-column strip (lane l: columns 4l..4l+3) and a slab of B bins.
// For every row it receives the four pixel bins of the lane packed in bytes and
// updates, per bin k and column j,
//     V[j][k] += L(y, k) + E_k(l) + P_k(j)
// where L is the count of k in the row left of the strip (carry table), E_k the count
// of k in lanes < l (one warp shuffle scan over four bins packed per word) and P_k(j)
// the count of k among the lane's columns <= j (byte-SIMD prefix of one-hot matches).
// V is then the unpadded integral-histogram value H(y+1, x+1, k) and leaves as one
// 16-byte streaming store per lane: each plane-row of the strip is a 512-byte run.
#pragma once

#include "spct_device.cuh"

namespace spct_dev {

// How the packed bins of a lane are formed (host-chosen, warp-uniform).
//   byte_mode: nbins <= 256 and the slab start is a multiple of 16; bytes hold the
//              absolute bin, and bin k0 + k (k0 % 16 == 0, k < 16) is matched as
//              (byte ^ k0) == k.
//              Columns past the image edge hold garbage: they only influence columns
//              further right, which are never stored.
//   otherwise: bytes hold bin - k0 for bins of the warp's slab and 0xFF elsewhere.
//   shift >= 0: gray uint8 with lo = 0, hi = 256 and nbins = 2^(8-shift): bin = v >> shift.
struct PixelMode {
    int byte_mode;
    int shift;
};

__host__ inline PixelMode make_pixel_mode(const QuantParams& q, int bin0) {
    PixelMode m{q.nbins <= 256 && bin0 % 16 == 0, -1};
    if (m.byte_mode && q.kind == SPCT_SRC_GRAY_U8 && q.fast_u8 && (q.nbins & (q.nbins - 1)) == 0) {
        int s = 8;
        while ((1 << (8 - s)) != q.nbins) --s;
        m.shift = s;
    }
    return m;
}

// Packed bins of pixels (x .. x+3, y).  x is a multiple of 4.
__device__ __forceinline__ uint32_t load_bins4(const QuantParams& q, const PixelMode& m, int x, int y, int k0, int nb) {
    if (m.shift >= 0) {
        const int64_t off = static_cast<int64_t>(y) * q.pitch + x;
        const uint8_t* p = static_cast<const uint8_t*>(q.p0) + off;
        uint32_t w;
        if (x + 3 < q.width && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
            w = __ldg(reinterpret_cast<const uint32_t*>(p));
        } else {
            w = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (x + j < q.width) w |= static_cast<uint32_t>(__ldg(p + j)) << (8 * j);
        }
        return (w >> m.shift) & (0x01010101u * (0xFFu >> m.shift));
    }
    if (m.byte_mode) {
        uint32_t w = 0;
        const bool full = x + 3 < q.width;
        if (full && q.kind == SPCT_SRC_GRAY_U8 &&
            ((reinterpret_cast<uintptr_t>(q.p0) + static_cast<int64_t>(y) * q.pitch + x) & 3) == 0) {
            const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(q.p0) +
                                                                        static_cast<int64_t>(y) * q.pitch + x));
#pragma unroll
            for (int j = 0; j < 4; ++j) w |= static_cast<uint32_t>(bin_of_u8((v >> (8 * j)) & 0xFFu, q)) << (8 * j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (x + j < q.width) w |= static_cast<uint32_t>(pixel_bin(q, x + j, y)) << (8 * j);
        }
        return w;
    }
    return load_rel4(q, x, y, k0, nb);
}

// Inclusive warp scan step with the shuffle's in-range predicate (no select).
__device__ __forceinline__ uint32_t scan_add(uint32_t v, int o) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
        "shfl.sync.up.b32 t|p, %1, %2, 0, 0xffffffff;\n\t"
        "@p add.u32 %1, %1, t;\n\t"
        "mov.u32 %0, %1;\n\t}"
        : "=r"(r), "+r"(v)
        : "r"(o));
    return r;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v = scan_add(v, o);
    return v;
}

template <int B>
__device__ __forceinline__ void vpart_init(uint32_t (&V)[4][B], const uint32_t* __restrict__ Hb, int band, int Lb,
                                           int kl0, int Wp, int x0) {
    if (band > 0 && Hb) {
        const uint32_t* hb = Hb + (static_cast<int64_t>(band - 1) * Lb + kl0) * Wp + x0;
#pragma unroll
        for (int k = 0; k < B; ++k) {
            uint4 v = *reinterpret_cast<const uint4*>(hb + static_cast<int64_t>(k) * Wp);
            V[0][k] = v.x;
            V[1][k] = v.y;
            V[2][k] = v.z;
            V[3][k] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < B; ++k) V[0][k] = V[1][k] = V[2][k] = V[3][k] = 0;
    }
}

// One row of the sweep.  `kpat0` = k0 * 0x01010101 in byte mode (k0 = global bin of
// the warp's first plane), 0 in relative mode.  `lt_row` points at L(y, kl0 ..) or is
// null for the first strip; `p` at column x0 of the warp's first plane in row y.
// GUARD: the slab has fewer than B live planes (k_live); `store`: lane inside the pitch.
template <int B, bool GUARD>
__device__ __forceinline__ void vpart_row(uint32_t (&V)[4][B], uint32_t bins4, uint32_t kpat0,
                                          const uint32_t* __restrict__ lt_row, uint32_t* p, int64_t plane_pitch,
                                          bool store, int k_live) {
#pragma unroll
    for (int g = 0; g < B / 4; ++g) {
        uint4 L = make_uint4(0, 0, 0, 0);
        if (lt_row) L = __ldg(reinterpret_cast<const uint4*>(lt_row) + g);
        uint32_t P[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            P[i] = match_prefix(bins4 ^ kpat0, 0x01010101u * static_cast<uint32_t>(4 * g + i));
        // lane totals (byte 3 of each prefix) -> one word, four bins
        const uint32_t packed = __byte_perm(__byte_perm(P[0], P[1], 0x0073), __byte_perm(P[2], P[3], 0x0073), 0x5410);
        const uint32_t excl = warp_incl_scan(packed) - packed;
        const uint32_t Lk[4] = {L.x, L.y, L.z, L.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = 4 * g + i;
            const uint32_t base = Lk[i] + __byte_perm(excl, 0, 0x4440 + i);
            V[0][k] += base + __byte_perm(P[i], 0, 0x4440);
            V[1][k] += base + __byte_perm(P[i], 0, 0x4441);
            V[2][k] += base + __byte_perm(P[i], 0, 0x4442);
            V[3][k] += base + (P[i] >> 24);
            st_cs_v4_pred(store && (!GUARD || k < k_live), p, V[0][k], V[1][k], V[2][k], V[3][k]);
            p += plane_pitch;
        }
    }
}

}  // namespace spct_dev

namespace spct_dev {

// One group of four planes (4g .. 4g+3) of vpart_row, for callers that interleave
// the row update with other work.  `p` points at plane 4g of the row.
template <int B>
__device__ __forceinline__ void vpart_group(uint32_t (&V)[4][B], int g, uint32_t dbins, uint4 L, uint32_t* p,
                                            int64_t plane_pitch, uint32_t store_mask) {
    // dbins = bins4 ^ kpat0; store_mask bit k: plane k is live and the lane is inside the pitch
    uint32_t P[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) P[i] = match_prefix(dbins, 0x01010101u * static_cast<uint32_t>(4 * g + i));
    const uint32_t packed = __byte_perm(__byte_perm(P[0], P[1], 0x0073), __byte_perm(P[2], P[3], 0x0073), 0x5410);
    const uint32_t excl = warp_incl_scan(packed) - packed;
    const uint32_t Lk[4] = {L.x, L.y, L.z, L.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
        const uint32_t base = Lk[i] + __byte_perm(excl, 0, 0x4440 + i);
        V[0][k] += base + __byte_perm(P[i], 0, 0x4440);
        V[1][k] += base + __byte_perm(P[i], 0, 0x4441);
        V[2][k] += base + __byte_perm(P[i], 0, 0x4442);
        V[3][k] += base + (P[i] >> 24);
        st_cs_v4_pred((store_mask >> k) & 1u, p, V[0][k], V[1][k], V[2][k], V[3][k]);
        p += plane_pitch;
    }
}

}  // namespace spct_dev

namespace spct_dev {

// Shift with PTX semantics: amounts >= 32 (including "negative" ones as unsigned) give 0.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t v, uint32_t n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(n));
    return r;
}

// Address of plane k of a row: prow + k * ppb bytes in one IMAD.WIDE (k * ppb < 2^32).
__device__ __forceinline__ uint32_t* plane_addr(uint32_t* prow, uint32_t k, uint32_t ppb) {
    uint64_t a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(k), "r"(ppb), "l"(reinterpret_cast<uint64_t>(prow)));
    return reinterpret_cast<uint32_t*>(a);
}

// 8 x (relative bin) of the lane's four columns, from dbins = bins4 ^ kpat0; a column off
// the warp's slab yields >= 128, so no group's one-hot shift lands inside a word.
__device__ __forceinline__ void onehot_shifts(uint32_t dbins, uint32_t (&t)[4]) {
    t[0] = (dbins & 0xFFu) << 3;
    t[1] = (dbins >> 5) & 0x7F8u;
    t[2] = (dbins >> 13) & 0x7F8u;
    t[3] = (dbins >> 21) & 0x7F8u;
}

// One group of four planes (4g .. 4g+3) of the row update, bin-major: Q[j] holds, in byte
// i, the count of bin 4g+i among the lane's columns <= j (the one-hot of column j is
// 1 << (8 r_j - 32 g)).  Q[3] is then already the packed per-lane total of the four bins
// that the cross-lane scan needs.  `p` points at plane 4g of the row.
template <int B>
__device__ __forceinline__ void vpart_group_q(uint32_t (&V)[4][B], int g, const uint32_t (&t)[4], uint4 L, uint32_t* p,
                                              int64_t plane_pitch, uint32_t store_mask) {
    uint32_t Q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t m = shl_clamp(1u, t[j] - 32u * g);
        Q[j] = j ? Q[j - 1] + m : m;
    }
    const uint32_t excl = warp_incl_scan(Q[3]) - Q[3];
    // bytes of Q + excl stay <= 128: the exclusive count folds in before the extraction
#pragma unroll
    for (int j = 0; j < 4; ++j) Q[j] += excl;
    const uint32_t Lk[4] = {L.x, L.y, L.z, L.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
        V[0][k] += Lk[i] + __byte_perm(Q[0], 0, 0x4440 + i);
        V[1][k] += Lk[i] + __byte_perm(Q[1], 0, 0x4440 + i);
        V[2][k] += Lk[i] + __byte_perm(Q[2], 0, 0x4440 + i);
        V[3][k] += Lk[i] + __byte_perm(Q[3], 0, 0x4440 + i);
        st_cs_v4_pred(store_mask & (1u << k), p, V[0][k], V[1][k], V[2][k], V[3][k]);
        p += plane_pitch;
    }
}

}  // namespace spct_dev
