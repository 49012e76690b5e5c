// Shared device-side pieces of the sm_100a integral-histogram path:
// the fused pixel -> bin stage (to_grayscale + quantize, reference
// imagecore.cpp:17-53) and small warp utilities.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "spct_cuda.h"

namespace spct_dev {

constexpr int kStrip = 128;  // columns per warp strip: 4 per lane -> one 512-B run per plane-row

// Quantisation parameters in the form the kernels consume.  `scale` is computed
// on the host exactly as the reference does (imagecore.cpp:33: bins / (hi - lo)).
struct QuantParams {
    int kind;        // SPCT_SRC_*
    int nbins;
    int fast_u8;     // 1: lo == 0, hi == 256 and uint8 input -> bin = (v * nbins) >> 8 (exact)
    double lo, scale;
    const void* p0;
    const void* p1;
    const void* p2;
    int64_t pitch;
    int width, height;
};

// floor + clamp of quantize_values (imagecore.cpp:35-38).  The reference converts
// floor(v) with static_cast<int>; on x86 an out-of-range or NaN double converts to
// INT_MIN, which the clamp then sends to bin 0.  CUDA's cvt saturates instead, so
// the out-of-range case is mapped explicitly to keep identical bins.
__device__ __forceinline__ int quantize_value(double v, const QuantParams& q) {
    double x = __dmul_rn(__dsub_rn(v, q.lo), q.scale);
    double f = floor(x);
    int b;
    if (f >= -2147483648.0 && f < 2147483648.0)
        b = static_cast<int>(f);
    else
        b = INT32_MIN;  // x86 cvttsd2si "integer indefinite"
    b = b < 0 ? 0 : b;
    b = b > q.nbins - 1 ? q.nbins - 1 : b;
    return b;
}

// Grayscale of one RGB pixel: lround((r+g+b)/3.0) == (r+g+b+1)/3 for every sum
// 0..765 (exhaustively checked in tests/test_oracle.py).
__device__ __forceinline__ uint32_t gray_of(uint32_t r, uint32_t g, uint32_t b) {
    return (r + g + b + 1u) / 3u;
}

__device__ __forceinline__ int bin_of_u8(uint32_t v, const QuantParams& q) {
    if (q.fast_u8) return static_cast<int>((v * static_cast<uint32_t>(q.nbins)) >> 8);
    return quantize_value(static_cast<double>(v), q);
}

// Global bin of pixel (x, y); x, y in range.
__device__ __forceinline__ int pixel_bin(const QuantParams& q, int x, int y) {
    const int64_t i = static_cast<int64_t>(y) * q.pitch + x;
    switch (q.kind) {
        case SPCT_SRC_BINS_U16:
            return static_cast<const uint16_t*>(q.p0)[i];
        case SPCT_SRC_GRAY_U8:
            return bin_of_u8(static_cast<const uint8_t*>(q.p0)[i], q);
        case SPCT_SRC_RGB_U8:
            return bin_of_u8(gray_of(static_cast<const uint8_t*>(q.p0)[i],
                                     static_cast<const uint8_t*>(q.p1)[i],
                                     static_cast<const uint8_t*>(q.p2)[i]),
                             q);
        default:
            return quantize_value(static_cast<const double*>(q.p0)[i], q);
    }
}

// Split form of pixel_bin for software pipelining: pixel_raw issues the load(s) and
// returns the raw value (u8 / u16 / packed RGB / f64 bits); bin_of_raw quantises it
// later, so the load latency overlaps a whole row of work.
__device__ __forceinline__ uint64_t pixel_raw(const QuantParams& q, int x, int y) {
    const int64_t i = static_cast<int64_t>(y) * q.pitch + x;
    switch (q.kind) {
        case SPCT_SRC_BINS_U16:
            return __ldg(static_cast<const uint16_t*>(q.p0) + i);
        case SPCT_SRC_GRAY_U8:
            return __ldg(static_cast<const uint8_t*>(q.p0) + i);
        case SPCT_SRC_RGB_U8:
            return static_cast<uint64_t>(__ldg(static_cast<const uint8_t*>(q.p0) + i)) |
                   (static_cast<uint64_t>(__ldg(static_cast<const uint8_t*>(q.p1) + i)) << 8) |
                   (static_cast<uint64_t>(__ldg(static_cast<const uint8_t*>(q.p2) + i)) << 16);
        default:
            return static_cast<uint64_t>(__double_as_longlong(__ldg(static_cast<const double*>(q.p0) + i)));
    }
}

__device__ __forceinline__ int bin_of_raw(uint64_t raw, const QuantParams& q) {
    switch (q.kind) {
        case SPCT_SRC_BINS_U16:
            return static_cast<int>(raw);
        case SPCT_SRC_GRAY_U8:
            return bin_of_u8(static_cast<uint32_t>(raw), q);
        case SPCT_SRC_RGB_U8:
            return bin_of_u8(gray_of(raw & 0xFF, (raw >> 8) & 0xFF, (raw >> 16) & 0xFF), q);
        default:
            return quantize_value(__longlong_as_double(static_cast<long long>(raw)), q);
    }
}

// Four consecutive pixels (x .. x+3) of row y as relative bins packed in bytes:
// byte j = bin(x+j) - k0 when it lies in [0, nb), else 0xFF (never matches).
// Columns >= width are 0xFF as well.  The aligned gray/bins fast paths issue one
// 32-/64-bit load per lane (a warp reads one contiguous 128/256-B segment).
__device__ __forceinline__ uint32_t load_rel4(const QuantParams& q, int x, int y, int k0, int nb) {
    int b[4];
    const int64_t row = static_cast<int64_t>(y) * q.pitch;
    const bool full = x + 3 < q.width;
    if (full && q.kind == SPCT_SRC_GRAY_U8 && ((reinterpret_cast<uintptr_t>(q.p0) + row + x) & 3) == 0) {
        uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(q.p0) + row + x));
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = bin_of_u8((w >> (8 * j)) & 0xFFu, q);
    } else if (full && q.kind == SPCT_SRC_BINS_U16 &&
               ((reinterpret_cast<uintptr_t>(q.p0) + 2 * (row + x)) & 7) == 0) {
        uint2 w = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(q.p0) + row + x));
        b[0] = w.x & 0xFFFFu;
        b[1] = w.x >> 16;
        b[2] = w.y & 0xFFFFu;
        b[3] = w.y >> 16;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = (x + j < q.width) ? pixel_bin(q, x + j, y) : -1;
    }
    uint32_t packed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int r = b[j] - k0;
        uint32_t byte = (b[j] >= 0 && static_cast<unsigned>(r) < static_cast<unsigned>(nb)) ? static_cast<uint32_t>(r) : 0xFFu;
        packed |= byte << (8 * j);
    }
    return packed;
}

// Bytes of `packed` equal to k -> 0x01, others 0x00 (exact: no cross-byte carries).
__device__ __forceinline__ uint32_t match_bytes(uint32_t packed, uint32_t kpat) {
    uint32_t x = packed ^ kpat;
    uint32_t t = ((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x;
    return (~t & 0x80808080u) >> 7;
}

// In-lane inclusive prefix of the one-hot matches in bytes: byte j = #{i <= j : byte_i == k}.
// Uses (j+1) - #non-matches: one IMAD folds the complement and the prefix multiply.
__device__ __forceinline__ uint32_t match_prefix(uint32_t packed, uint32_t kpat) {
    const uint32_t x = packed ^ kpat;
    const uint32_t nz = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;  // 0x80 where byte != k
    return 0x04030201u - (nz >> 7) * 0x01010101u;
}

// 16-byte streaming store under a predicate (the address is computed unconditionally by
// the caller so the compiler emits a predicated STG rather than a branch).
__device__ __forceinline__ void st_cs_v4_if(bool pred, uint32_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    if (pred) __stcs(reinterpret_cast<uint4*>(p), make_uint4(a, b, c, d));
}

// Same store, predicated in PTX so it never becomes a branch.  No "memory" clobber:
// nothing in the sweeps reads the integral histogram back, and a clobber would pin
// every shared-memory access around the store.
__device__ __forceinline__ void st_cs_v4_pred(uint32_t pred, uint32_t* p, uint32_t a, uint32_t b, uint32_t c,
                                              uint32_t d) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
        "@q st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
        "r"(a), "r"(b), "r"(c), "r"(d), "r"(pred));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace spct_dev
