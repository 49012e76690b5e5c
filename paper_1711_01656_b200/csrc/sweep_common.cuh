// The per-row integral-histogram update shared by the build sweep and the fused
// build+match sweep.
//
// A warp owns a 128-column strip (lane l: columns 4l..4l+3) and a slab of B bins.
// For every row it receives the row's four relative bins per lane packed in bytes
// (0xFF = not in the slab) and updates, per bin k and column j,
//     V[j][k] += L(y, k) + E_k(l) + P_k(j)
// where L is the count of k in the row left of the strip (carry table), E_k the count
// of k in lanes < l (one warp shuffle scan over four bins packed per word) and P_k(j)
// the count of k among the lane's columns <= j (byte-SIMD prefix of one-hot matches).
// V is then the unpadded integral-histogram value H(y+1, x+1, k) and leaves as one
// 16-byte streaming store per lane: each plane-row of the strip is a 512-byte run.
#pragma once

#include "spct_device.cuh"

namespace spct_dev {

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

// One row of the sweep.  `lt_row` points at L(y, kl0 .. kl0+B) (16-byte aligned) or is
// null for the first strip; `rowp` at column x0 of plane kl0, row y; stores go to
// rowp + k*plane_pitch when `store` and k < k_live.
template <int B>
__device__ __forceinline__ void vpart_row(uint32_t (&V)[4][B], uint32_t cur, const uint32_t* __restrict__ lt_row,
                                          int lane, uint32_t* rowp, int64_t plane_pitch, bool store, int k_live) {
#pragma unroll
    for (int g = 0; g < B / 4; ++g) {
        uint4 L = make_uint4(0, 0, 0, 0);
        if (lt_row) L = __ldg(reinterpret_cast<const uint4*>(lt_row) + g);
        uint32_t P[4];
        uint32_t packed = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t k = 4 * g + i;
            P[i] = match_bytes(cur, 0x01010101u * k) * 0x01010101u;
            packed |= (P[i] >> 24) << (8 * i);
        }
        uint32_t v = packed;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        const uint32_t excl = v - packed;
        const uint32_t Lk[4] = {L.x, L.y, L.z, L.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = 4 * g + i;
            const uint32_t base = Lk[i] + ((excl >> (8 * i)) & 0xFFu);
            V[0][k] += base + (P[i] & 0xFFu);
            V[1][k] += base + ((P[i] >> 8) & 0xFFu);
            V[2][k] += base + ((P[i] >> 16) & 0xFFu);
            V[3][k] += base + (P[i] >> 24);
            if (store && k < k_live)
                __stcs(reinterpret_cast<uint4*>(rowp + static_cast<int64_t>(k) * plane_pitch),
                       make_uint4(V[0][k], V[1][k], V[2][k], V[3][k]));
        }
    }
}

}  // namespace spct_dev
