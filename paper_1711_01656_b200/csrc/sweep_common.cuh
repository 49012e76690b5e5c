// The per-row integral-histogram update shared by the build sweep and the fused
// build+match sweep.
//
// A warp owns a 128-column strip (lane l: columns 4l..4l+3) and a slab of B bins.
// For every row it receives the four pixel bins of the lane packed in bytes and
// updates, per bin k and column j,
//     V[j][k] += L(y, k) + E_k(l) + P_k(j)
// where L is the count of k in the row left of the strip (carry table), E_k the count
// of k in lanes < l (one warp shuffle scan over four bins packed per word) and P_k(j)
// the count of k among the lane's columns <= j (one-hot shifts, vpart_group_q).
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

// load_bins4 split in two for the gray shift mode, so a row-ahead prefetch keeps only the
// raw load in flight and the decode sits at the consumer (the shift would otherwise
// wait on the load right where it is issued).
__device__ __forceinline__ uint32_t load_bins4_raw(const QuantParams& q, const PixelMode& m, int x, int y, int k0,
                                                   int nb) {
    if (m.shift < 0) return load_bins4(q, m, x, y, k0, nb);
    const int64_t off = static_cast<int64_t>(y) * q.pitch + x;
    const uint8_t* p = static_cast<const uint8_t*>(q.p0) + off;
    if (x + 3 < q.width && (reinterpret_cast<uintptr_t>(p) & 3) == 0) return __ldg(reinterpret_cast<const uint32_t*>(p));
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (x + j < q.width) w |= static_cast<uint32_t>(__ldg(p + j)) << (8 * j);
    return w;
}

__device__ __forceinline__ uint32_t decode_bins4(const PixelMode& m, uint32_t raw) {
    return m.shift < 0 ? raw : (raw >> m.shift) & (0x01010101u * (0xFFu >> m.shift));
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

}  // namespace spct_dev

namespace spct_dev {

// Shift with PTX semantics: amounts >= 32 (including "negative" ones as unsigned) give 0.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t v, uint32_t n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(n));
    return r;
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
// MODE 0 stores the row; 1 / 2 add / subtract it into the tensor already there (the joint
// integral histogram of a frame window, motion.cpp:51-60).
// `pre` (MODE 1 / 2): the group's four tensor cells of this row, loaded a row ahead.
template <int B, int MODE = 0>
__device__ __forceinline__ void vpart_group_q(uint32_t (&V)[4][B], int g, const uint32_t (&t)[4], uint4 L, uint32_t* p,
                                              int64_t plane_pitch, uint32_t store_mask, const uint4* pre = nullptr) {
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
        if (MODE == 0) {
            st_cs_v4_pred(store_mask & (1u << k), p, V[0][k], V[1][k], V[2][k], V[3][k]);
        } else if (store_mask & (1u << k)) {
            uint4 o = pre ? pre[i] : *reinterpret_cast<const uint4*>(p);
            if (MODE == 1) o = make_uint4(o.x + V[0][k], o.y + V[1][k], o.z + V[2][k], o.w + V[3][k]);
            else o = make_uint4(o.x - V[0][k], o.y - V[1][k], o.z - V[2][k], o.w - V[3][k]);
            *reinterpret_cast<uint4*>(p) = o;
        }
        p += plane_pitch;
    }
}

}  // namespace spct_dev

namespace spct_dev {

// V at the top of a band (the unpadded IH row y0 - 1) from the carry tables of
// carries.cu: H(y0, x + 1, k) = A[k][band-1][strip] (rows < y0, columns left of the strip)
// + the inclusive prefix along the strip of C[band-1][k][x] (column counts above y0).
// Lane l owns columns x0 .. x0+3 of the strip; kl0 is the warp's first slab-local bin.
template <int B>
__device__ __forceinline__ void vpart_init_ca(uint32_t (&V)[4][B], const uint16_t* __restrict__ C,
                                              const uint32_t* __restrict__ A, int band, int strip, int nbands,
                                              int nstrips, int Lb, int Wp, int kl0, int x0) {
    if (band > 0 && C) {
        const uint16_t* cb = C + (static_cast<int64_t>(band - 1) * Lb + kl0) * Wp + x0;
        const uint32_t* ab = A + (static_cast<int64_t>(kl0) * (nbands - 1) + band - 1) * nstrips + strip;
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const uint2 c = *reinterpret_cast<const uint2*>(cb + static_cast<int64_t>(k) * Wp);
            const uint32_t p0 = c.x & 0xFFFFu, p1 = p0 + (c.x >> 16), p2 = p1 + (c.y & 0xFFFFu), p3 = p2 + (c.y >> 16);
            const uint32_t base = __ldg(ab + static_cast<int64_t>(k) * (nbands - 1) * nstrips) + warp_incl_scan(p3) - p3;
            V[0][k] = base + p0;
            V[1][k] = base + p1;
            V[2][k] = base + p2;
            V[3][k] = base + p3;
        }
    } else {
#pragma unroll
        for (int k = 0; k < B; ++k) V[0][k] = V[1][k] = V[2][k] = V[3][k] = 0;
    }
}

// Row carries of a warp's B-bin slab (B / 2 words of u16 pairs per row), fetched as one
// coalesced load of 64 / B rows per lane-word and one chunk ahead, so the L2 latency of
// the carry table never sits on a row's critical path; row r of the chunk is read back
// with shuffles.  `p` is row 0's carries of the warp's first bin (null: first strip).
template <int B>
struct LtRows {
    static constexpr int kWords = B / 2;          // words per row
    static constexpr int kRows = 32 / kWords;     // rows per chunk
    const uint16_t* p;
    int Lb, nrows;
    uint32_t cur = 0, nxt = 0;
    __device__ __forceinline__ uint32_t fetch(int r0) const {
        const int l = static_cast<int>(threadIdx.x & 31);
        const int r = r0 + l / kWords;
        return (p && r < nrows) ? __ldg(reinterpret_cast<const uint32_t*>(p + static_cast<int64_t>(r) * Lb) + l % kWords)
                                : 0u;
    }
    __device__ __forceinline__ void start() { nxt = fetch(0); }
    // call once per row r = 0, 1, ... before group()
    __device__ __forceinline__ void row(int r) {
        if (r % kRows == 0) {
            cur = nxt;
            nxt = fetch(r + kRows);
        }
    }
    __device__ __forceinline__ uint4 group(int r, int g) const {
        const int sl = (r % kRows) * kWords + 2 * g;
        const uint32_t a = __shfl_sync(0xffffffffu, cur, sl), b = __shfl_sync(0xffffffffu, cur, sl + 1);
        return make_uint4(a & 0xFFFFu, a >> 16, b & 0xFFFFu, b >> 16);
    }
};

// Row carries of group g (4 bins) from a u16 carry row (null: first strip, all zero).
__device__ __forceinline__ uint4 lt16_group(const uint16_t* lt_row, int g) {
    if (!lt_row) return make_uint4(0, 0, 0, 0);
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(lt_row) + g);
    return make_uint4(v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16);
}

}  // namespace spct_dev
