#include <type_traits>

#include "spct_internal.h"

using namespace spct_dev;

// Carry tables of the banded sweeps.
//
// The build sweep (ih_build.cu) and the fused build+match sweep (fused_kernel.cuh) start
// each (strip s, band j) tile from
//   Lt16[s][y][kl] = count of kl in row y, columns [0, 128 s)                    (u16)
//   C16[j-1][kl][x] = count of kl in column x, rows < y0_j                       (u16)
//   A32[kl][j-1][s] = count of kl in rows < y0_j, columns [0, 128 s)             (u32)
// and rebuilds H(y0_j, x, kl) = A + sum over the strip's columns <= x of C16 itself, so
// no 32-bit band-carry table is written or read.  Two passes over 1 B/px:
//   fcarry_tiles_kernel   one CTA per (strip, band, 128-bin chunk): the strip-row
//                         histograms (u8), the band's column counts and band x strip totals;
//   fcarry_prefix_kernel  prefix of the strip-row histograms over strips (-> Lt16), of the
//                         column counts over bands (in place -> C16), and one CTA per bin
//                         for the 2-D prefix of the band x strip totals (-> A32).

namespace spct_carry {

constexpr int kTileBins = 128;
using spct_impl::kMaxCarryCh;

// The carry tables of up to kMaxCarryCh same-shape sources (the channels of a tracking
// batch) in one launch of each kernel: grid.z (tiles) / grid.y (prefix) selects the source.
struct CarryBatch {
    QuantParams q[kMaxCarryCh];
    uint8_t* R8[kMaxCarryCh];
    uint16_t* C16[kMaxCarryCh];
    uint32_t* T1[kMaxCarryCh];
    uint16_t* S16[kMaxCarryCh];
    uint16_t* Lt16[kMaxCarryCh];
    int nchunk;  // 128-bin chunks per source (grid.z = sources x chunks)
};

template <bool G8>
__global__ void __launch_bounds__(256) fcarry_tiles_kernel(const __grid_constant__ CarryBatch cb, int bin0, int bins,
                                                           int Lb, int nstrips, int nbands, int band_rows, int tb,
                                                           int suf_row0) {
    const int ch = blockIdx.z / cb.nchunk;
    const QuantParams& q = cb.q[ch];
    uint8_t* __restrict__ R8 = cb.R8[ch];
    uint16_t* __restrict__ C16 = cb.C16[ch];
    uint32_t* __restrict__ T1 = cb.T1[ch];
    uint16_t* __restrict__ S16 = cb.S16[ch];
    // column counts as u16 pairs (a column's count within a band is < 2^16, as in C16):
    // word h * 32 + lane of a bin row holds strip columns 4 lane + 2h (low) and + 2h + 1
    // (high), i.e. already the C16 layout; half the shared memory of u32 counters, so a
    // whole grid of tiles is resident in one wave
    extern __shared__ uint32_t fsm[];
    uint32_t* cnt = fsm;                     // [tb bins][64 words]
    uint32_t* rh = fsm + tb * kStrip / 2;    // [8 warps][128 bins]
    uint32_t* cs = rh + 8 * kTileBins;       // [tb bins][64 words]: window-start suffix counts
    const int s = blockIdx.x, j = blockIdx.y, kc0 = (blockIdx.z % cb.nchunk) * kTileBins;
    const int kcn = min(kTileBins, Lb - kc0);
    const bool need_r = s + 1 < nstrips, need_c = j + 1 < nbands;
    const bool need_s = need_c && S16;
    if (!need_r && !need_c) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // (16-byte clears: every region is a multiple of 4 words and 16-byte aligned)
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    if (need_c)
        for (int i = tid; i < tb * kStrip / 8; i += 256) reinterpret_cast<uint4*>(cnt)[i] = z4;
    if (need_s)
        for (int i = tid; i < tb * kStrip / 8; i += 256) reinterpret_cast<uint4*>(cs)[i] = z4;
    for (int i = tid; i < 2 * kTileBins; i += 256) reinterpret_cast<uint4*>(rh)[i] = z4;
    __syncthreads();
    const int y0 = j * band_rows, y1 = min(q.height, y0 + band_rows);
    const int ys = y0 + suf_row0;  // the suffix rows [ys, y1)
    const int x = s * kStrip + 4 * lane;
    const int klo = bin0 + kc0, khi = min(kcn, bins - kc0);
    uint32_t* rw = rh + warp * kTileBins;
    // column 4 lane + c of the strip is counted in word (c >> 1) * 32 + lane, half c & 1
    // (conflict-free atomics)
    // 8-bit gray with the default range: four pixels per 32-bit load (per source: a batch
    // may mix them with BinMaps)
    const bool wide = G8 && q.kind == SPCT_SRC_GRAY_U8 && q.fast_u8 && x + 3 < q.width &&
                      ((reinterpret_cast<uintptr_t>(q.p0) + x) & 3) == 0 && (q.pitch & 3) == 0;
    // a uint16 BinMap (the orientation channel): four bins per 8-byte load
    const bool wide16 = !G8 && q.kind == SPCT_SRC_BINS_U16 && x + 3 < q.width &&
                        ((reinterpret_cast<uintptr_t>(q.p0) + 2 * static_cast<uintptr_t>(x)) & 7) == 0 && (q.pitch & 3) == 0;
    auto bins4 = [&](int y, uint2 w, int (&b)[4]) {
        if (wide) {
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = static_cast<int>((((w.x >> (8 * c)) & 0xFFu) * q.nbins) >> 8);
        } else if (wide16) {
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = static_cast<int>(((c < 2 ? w.x : w.y) >> (16 * (c & 1))) & 0xFFFFu);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = x + c < q.width ? pixel_bin(q, x + c, y) : -1;
        }
    };
    // every bin of the source lands in this chunk (one chunk, the whole histogram): no
    // per-pixel range check
    const bool full_range = wide && klo == 0 && khi >= q.nbins;
    uint8_t* const r8col = R8 + static_cast<int64_t>(s) * q.height * Lb + kc0 + 4 * lane;
    auto count_row = [&](int y, const int (&b)[4], auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int k = b[c] - klo;
            if (FULL || (b[c] >= 0 && static_cast<unsigned>(k) < static_cast<unsigned>(khi))) {
                if (need_c) atomicAdd(&cnt[k * (kStrip / 2) + (c >> 1) * 32 + lane], 1u << (16 * (c & 1)));
                if (need_s && y >= ys) atomicAdd(&cs[k * (kStrip / 2) + (c >> 1) * 32 + lane], 1u << (16 * (c & 1)));
                if (need_r) atomicAdd(&rw[k], 1u);
            }
        }
        if (need_r) {
            __syncwarp();
            if (4 * lane < kcn) {
                const uint4 h = *reinterpret_cast<const uint4*>(rw + 4 * lane);
                *reinterpret_cast<uint4*>(rw + 4 * lane) = make_uint4(0, 0, 0, 0);
                const uint32_t packed = h.x | (h.y << 8) | (h.z << 16) | (h.w << 24);
                *reinterpret_cast<uint32_t*>(r8col + static_cast<int64_t>(y) * Lb) = packed;
            }
            __syncwarp();
        }
    };
    // rows y0 + warp + 8 i; the 8-bit gray words of four rows are loaded before any is counted
    const uint8_t* colp = static_cast<const uint8_t*>(q.p0) + x;
    const uint16_t* colp16 = static_cast<const uint16_t*>(q.p0) + x;
    auto rows = [&](auto full_tag) {
        int y = y0 + warp;
        for (; y + 24 < y1; y += 32) {
            uint2 w[4] = {};
            if (wide) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    w[u].x = __ldg(reinterpret_cast<const uint32_t*>(colp + static_cast<int64_t>(y + 8 * u) * q.pitch));
            } else if (wide16) {
#pragma unroll
                for (int u = 0; u < 4; ++u) w[u] = __ldg(reinterpret_cast<const uint2*>(colp16 + static_cast<int64_t>(y + 8 * u) * q.pitch));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                int b[4];
                bins4(y + 8 * u, w[u], b);
                count_row(y + 8 * u, b, full_tag);
            }
        }
        for (; y < y1; y += 8) {
            uint2 w = {};
            if (wide) w.x = __ldg(reinterpret_cast<const uint32_t*>(colp + static_cast<int64_t>(y) * q.pitch));
            else if (wide16) w = __ldg(reinterpret_cast<const uint2*>(colp16 + static_cast<int64_t>(y) * q.pitch));
            int b[4];
            bins4(y, w, b);
            count_row(y, b, full_tag);
        }
    };
    if (full_range)
        rows(std::true_type{});
    else
        rows(std::false_type{});
    if (!need_c) return;
    __syncthreads();
    const int Wp = nstrips * kStrip;
    // warp w dumps bins w, w + 8, ...: lane l the columns 4 l .. 4 l + 3 of the C16 (and S16)
    // rows, and the warp's sum of the bin's column counts is its band x strip total,
    // [kl][j][s] (one REDUX)
    const int64_t o0 = (static_cast<int64_t>(j) * Lb + kc0 + warp) * Wp + s * kStrip + 4 * lane, ostep = 8 * static_cast<int64_t>(Wp);
    uint32_t* t1 = T1 + (static_cast<int64_t>(kc0 + warp) * (nbands - 1) + j) * nstrips + s;
    const int64_t tstep = 8 * static_cast<int64_t>(nbands - 1) * nstrips;
    for (int k = warp, i = 0; k < kcn; k += 8, ++i) {
        const uint32_t* ck = cnt + k * (kStrip / 2) + lane;
        const uint32_t p0 = ck[0], p1 = ck[32];
        const int64_t o = o0 + i * ostep;
        *reinterpret_cast<uint2*>(C16 + o) = make_uint2(p0, p1);
        if (need_s) {
            const uint32_t* cq = cs + k * (kStrip / 2) + lane;
            *reinterpret_cast<uint2*>(S16 + o) = make_uint2(cq[0], cq[32]);
        }
        const uint32_t t = __reduce_add_sync(0xffffffffu, (p0 & 0xFFFFu) + (p0 >> 16) + (p1 & 0xFFFFu) + (p1 >> 16));
        if (lane == 0) t1[i * tstep] = t;
    }
}

// Blocks [0, nb_lt): row carries (thread = (row, 4 bins)); blocks [nb_lt, ...): column
// counts over bands (thread = (bin, 4 columns)), in place.
// ... and blocks [nb_lt + nb_c, + Lb): the corner sums of one bin each (corner_block).
__device__ void corner_block(int kl, int nstrips, int nbands, uint32_t* __restrict__ T1, uint32_t* tsm);

__global__ void __launch_bounds__(256) fcarry_prefix_kernel(const __grid_constant__ CarryBatch cb, int H, int Lb, int Wp,
                                                            int nstrips, int nbands, int nb_lt, int nb_c) {
    extern __shared__ uint32_t corner_sm[];
    const uint8_t* __restrict__ R8 = cb.R8[blockIdx.y];
    uint16_t* __restrict__ Lt16 = cb.Lt16[blockIdx.y];
    uint16_t* __restrict__ C16 = cb.C16[blockIdx.y];
    uint32_t* __restrict__ A32 = cb.T1[blockIdx.y];
    if (static_cast<int>(blockIdx.x) >= nb_lt + nb_c) {
        corner_block(static_cast<int>(blockIdx.x) - nb_lt - nb_c, nstrips, nbands, A32, corner_sm);
        return;
    }
    if (static_cast<int>(blockIdx.x) < nb_lt) {
        const int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;  // (y, quad)
        const int quads = Lb / 4;
        if (i >= static_cast<int64_t>(H) * quads) return;
        const int64_t off = (i / quads) * Lb + 4 * (i % quads);
        const int64_t sstride = static_cast<int64_t>(H) * Lb;
        uint32_t a0 = 0, a1 = 0;  // u16 pairs: bins {0,1}, {2,3}
        constexpr int U = 8;       // loads in flight
        for (int s0 = 0; s0 + 1 < nstrips; s0 += U) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                v[u] = s0 + u + 1 < nstrips ? __ldg(reinterpret_cast<const uint32_t*>(R8 + (s0 + u) * sstride + off)) : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (s0 + u + 1 >= nstrips) break;
                a0 += __byte_perm(v[u], 0, 0x4140);  // {b0, b1} as u16 pair
                a1 += __byte_perm(v[u], 0, 0x4342);
                *reinterpret_cast<uint2*>(Lt16 + (s0 + u + 1) * sstride + off) = make_uint2(a0, a1);
            }
        }
    } else {
        const int64_t i = static_cast<int64_t>(blockIdx.x - nb_lt) * 256 + threadIdx.x;  // (bin, quad)
        const int64_t plane = static_cast<int64_t>(Lb) * Wp;
        if (i >= plane / 4) return;
        uint16_t* p = C16 + 4 * i;
        uint2 acc = make_uint2(0, 0);
        constexpr int U = 8;  // loads in flight; the next group is loaded before this one is
                              // stored (in place: the loads could not move past the stores)
        auto load = [&](int j0, uint2 (&v)[U]) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                v[u] = j0 + u + 1 < nbands ? *reinterpret_cast<const uint2*>(p + (j0 + u) * plane) : make_uint2(0, 0);
        };
        uint2 cur[U], nxt[U];
        load(0, cur);
        for (int j0 = 0; j0 + 1 < nbands; j0 += U) {
            if (j0 + U + 1 < nbands) load(j0 + U, nxt);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (j0 + u + 1 >= nbands) break;
                acc.x += cur[u].x;  // u16 pairs: column counts stay below 2^16 (H < 65536)
                acc.y += cur[u].y;
                *reinterpret_cast<uint2*>(p + (j0 + u) * plane) = acc;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = nxt[u];
        }
    }
}

// One CTA per bin: A[kl][j][s] = sum_{j' <= j} sum_{s' < s} T1[kl][j'][s'], in place.
__device__ void corner_block(int kl, int nstrips, int nbands, uint32_t* __restrict__ T1, uint32_t* tsm) {
    const int J = nbands - 1, S = nstrips;
    uint32_t* t = T1 + static_cast<int64_t>(kl) * J * S;
    for (int i = threadIdx.x; i < J * S; i += blockDim.x) tsm[i] = t[i];
    __syncthreads();
    for (int jj = threadIdx.x; jj < J; jj += blockDim.x) {  // exclusive prefix over strips
        uint32_t run = 0;
        for (int s = 0; s < S; ++s) {
            const uint32_t v = tsm[jj * S + s];
            tsm[jj * S + s] = run;
            run += v;
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x) {  // inclusive prefix over bands
        uint32_t run = 0;
        for (int jj = 0; jj < J; ++jj) {
            run += tsm[jj * S + s];
            t[jj * S + s] = run;
        }
    }
}

}  // namespace spct_carry

namespace spct_impl {

using namespace spct_carry;

FusedCarryLayout fused_carry_layout(const BuildPlan& p, int height, bool window) {
    FusedCarryLayout L{};
    const size_t lb = static_cast<size_t>(p.Lb);
    L.lt_off = 0;
    L.lt_bytes = p.nstrips > 1 ? round_up(static_cast<int64_t>(p.nstrips) * height * lb * 2, 256) : 0;
    L.r_off = L.lt_off + L.lt_bytes;
    L.r_bytes = p.nstrips > 1 ? round_up(static_cast<int64_t>(p.nstrips - 1) * height * lb, 256) : 0;
    L.c_off = L.r_off + L.r_bytes;
    L.c_bytes = p.nbands > 1 ? round_up(static_cast<int64_t>(p.nbands - 1) * lb * p.Wp * 2, 256) : 0;
    L.a_off = L.c_off + L.c_bytes;
    L.a_bytes = p.nbands > 1 ? round_up(static_cast<int64_t>(p.nbands - 1) * p.nstrips * lb * 4, 256) : 0;
    L.s_off = L.a_off + L.a_bytes;
    L.s_bytes = window ? L.c_bytes : 0;
    L.total = L.s_off + L.s_bytes;
    return L;
}

spct_status build_fused_carries_multi(int n, const QuantParams* qs, const spct_ih& out, const BuildPlan& p,
                                      void* const* workspaces, size_t ws_bytes, cudaStream_t s, FusedCarries* fcs,
                                      int kh) {
    if (n < 1 || n > kMaxCarryCh) return contract("ih_build_match: 1 .. 8 sources per batch");
    const FusedCarryLayout L = fused_carry_layout(p, out.height, kh > 1);
    for (int c = 0; c < n; ++c) fcs[c] = FusedCarries{};
    if (L.total == 0) return SPCT_OK;
    CarryBatch cb{};
    cb.nchunk = static_cast<int>(ceil_div(p.Lb, kTileBins));
    bool g8 = false;  // some source is 8-bit gray: the kernel variant with the 4-pixel loads
    for (int c = 0; c < n; ++c) {
        if (!workspaces[c] || ws_bytes < L.total)
            return contract("ih_build_match: workspace too small (query spct_cu_ih_build_workspace)");
        char* ws = static_cast<char*>(workspaces[c]);
        cb.q[c] = qs[c];
        cb.R8[c] = L.r_bytes ? reinterpret_cast<uint8_t*>(ws + L.r_off) : nullptr;
        cb.Lt16[c] = L.lt_bytes ? reinterpret_cast<uint16_t*>(ws + L.lt_off) : nullptr;
        cb.C16[c] = L.c_bytes ? reinterpret_cast<uint16_t*>(ws + L.c_off) : nullptr;
        cb.T1[c] = L.a_bytes ? reinterpret_cast<uint32_t*>(ws + L.a_off) : nullptr;
        cb.S16[c] = L.s_bytes ? reinterpret_cast<uint16_t*>(ws + L.s_off) : nullptr;
        g8 = g8 || (qs[c].kind == SPCT_SRC_GRAY_U8 && qs[c].fast_u8);
    }
    // window-start rows in every band: [y0 + o, y1), o = (-(kh - 1)) mod band_rows
    const int suf_row0 = kh > 1 ? (p.band_rows - (kh - 1) % p.band_rows) % p.band_rows : 0;
    const int tb = std::min(p.Lb, kTileBins);
    const size_t smem = (static_cast<size_t>(tb) * (kStrip / 2) * (L.s_bytes ? 2 : 1) + 8 * kTileBins) * 4;
    ensure_smem(fcarry_tiles_kernel<true>, smem);
    ensure_smem(fcarry_tiles_kernel<false>, smem);
    dim3 g(p.nstrips, p.nbands, static_cast<unsigned>(cb.nchunk * n));
    if (g8)
        fcarry_tiles_kernel<true><<<g, 256, smem, s>>>(cb, out.bin0, out.bins, p.Lb, p.nstrips, p.nbands, p.band_rows, tb,
                                                        suf_row0);
    else
        fcarry_tiles_kernel<false><<<g, 256, smem, s>>>(cb, out.bin0, out.bins, p.Lb, p.nstrips, p.nbands, p.band_rows,
                                                         tb, suf_row0);
    if (auto st = launch_status("fcarry_tiles_kernel")) return st;
    const int nb_lt = L.lt_bytes ? static_cast<int>(ceil_div(static_cast<int64_t>(out.height) * (p.Lb / 4), 256)) : 0;
    const int nb_c = L.c_bytes ? static_cast<int>(ceil_div(static_cast<int64_t>(p.Lb) * p.Wp / 4, 256)) : 0;
    const int nb_a = L.a_bytes ? p.Lb : 0;
    const size_t tsm = L.a_bytes ? static_cast<size_t>(p.nbands - 1) * p.nstrips * 4 : 0;
    if (tsm > 200 * 1024) return contract("ih_build_match: image too large for the fused carry tables");
    if (nb_lt + nb_c + nb_a > 0) {
        ensure_smem(fcarry_prefix_kernel, tsm);
        fcarry_prefix_kernel<<<dim3(nb_lt + nb_c + nb_a, n), 256, tsm, s>>>(cb, out.height, p.Lb, p.Wp, p.nstrips,
                                                                          p.nbands, nb_lt, nb_c);
        if (auto st = launch_status("fcarry_prefix_kernel")) return st;
    }
    for (int c = 0; c < n; ++c) {
        fcs[c].Lt = cb.Lt16[c];
        fcs[c].C = cb.C16[c];
        fcs[c].A = cb.T1[c];
        fcs[c].S = cb.S16[c];
    }
    return SPCT_OK;
}

spct_status build_fused_carries(const QuantParams& q, const spct_ih& out, const BuildPlan& p, void* workspace,
                                size_t ws_bytes, cudaStream_t s, FusedCarries* fc, int kh) {
    void* ws[1] = {workspace};
    return build_fused_carries_multi(1, &q, out, p, ws, ws_bytes, s, fc, kh);
}

}  // namespace spct_impl
