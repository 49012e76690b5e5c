// IHT1 wire format of an integral-histogram tensor.
//
// Reference: integral.hpp:132-135, dump_tensor / load_tensor integral.cpp:619-659:
//   "IHT1", little-endian u32 bins, height, width, elem_bytes (= 8), then the planes in
//   storage order (plane-major, row-major, zero padding row / column) as little-endian u64.
// Here the tensor lives in HBM as unpadded uint32; a dump streams it out in row chunks
// (device kernel widens to the padded file layout, pinned double buffer, overlapped
// D2H + fwrite) and a load streams it back in (fread into pinned memory, H2D, device
// kernel narrows and checks).  elem_bytes = 4 is accepted as an extension (half the bytes;
// the reference loader rejects it, so dumps default to 8).  Errors follow the reference:
// SPCT_ERR_IO with its messages, contract errors for descriptor mismatches.
#include <cstdio>
#include <cstring>
#include <string>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_iht1 {

constexpr int64_t kChunkBytes = 32ll << 20;  // per staging buffer

// Padded rows [r0, r1) of plane k (padded row r = IH row r, row 0 zero) -> file bytes.
template <typename E>
__global__ void widen_rows_kernel(spct_ih t, int k, int r0, int r1, E* __restrict__ dst) {
    const int64_t W1 = t.width + 1;
    const int64_t n = static_cast<int64_t>(r1 - r0) * W1;
    const uint32_t* plane = t.data + static_cast<int64_t>(k) * t.plane_pitch;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t y = r0 + i / W1, x = i % W1;
        dst[i] = (y > 0 && x > 0) ? static_cast<E>(plane[(y - 1) * t.row_pitch + (x - 1)]) : E(0);
    }
}

// File bytes of padded rows [r0, r1) of plane k -> the tensor; flags: bit 0 nonzero
// padding, bit 1 a value above 2^32 - 1 (neither is representable in the device layout).
template <typename E>
__global__ void narrow_rows_kernel(spct_ih t, int k, int r0, int r1, const E* __restrict__ src,
                                   unsigned* __restrict__ flags) {
    const int64_t W1 = t.width + 1;
    const int64_t n = static_cast<int64_t>(r1 - r0) * W1;
    uint32_t* plane = t.data + static_cast<int64_t>(k) * t.plane_pitch;
    unsigned bad = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t y = r0 + i / W1, x = i % W1;
        const uint64_t v = static_cast<uint64_t>(src[i]);
        if (y == 0 || x == 0) {
            if (v) bad |= 1u;
        } else {
            if (v >> 32) bad |= 2u;
            plane[(y - 1) * t.row_pitch + (x - 1)] = static_cast<uint32_t>(v);
        }
    }
    if (bad) atomicOr(flags, bad);
}

int grid_n(int64_t n) { return static_cast<int>(std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 16)); }

spct_status io(const std::string& msg) {
    set_error(msg);
    return SPCT_ERR_IO;
}

struct Staging {  // two pinned host buffers + two device buffers + events
    void* host[2] = {nullptr, nullptr};
    void* dev[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Staging() {
        for (int i = 0; i < 2; ++i) {
            if (host[i]) cudaFreeHost(host[i]);
            if (dev[i]) cudaFree(dev[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
    }
    spct_status init(size_t bytes) {
        for (int i = 0; i < 2; ++i) {
            if (auto st = cuda_status(cudaHostAlloc(&host[i], bytes, cudaHostAllocDefault), "IHT1 pinned buffer")) return st;
            if (auto st = cuda_status(cudaMalloc(&dev[i], bytes), "IHT1 device buffer")) return st;
            if (auto st = cuda_status(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "IHT1 event")) return st;
        }
        return SPCT_OK;
    }
};

// Row chunks of the padded tensor: (plane, r0, r1) in file order.
template <typename F>
spct_status for_chunks(const spct_ih& t, int elem, F&& f) {
    const int64_t row_bytes = static_cast<int64_t>(t.width + 1) * elem;
    const int rows = static_cast<int>(std::max<int64_t>(1, kChunkBytes / row_bytes));
    int i = 0;
    for (int k = 0; k < t.bins; ++k)
        for (int r0 = 0; r0 <= t.height; r0 += rows, ++i)
            if (auto st = f(i, k, r0, std::min(t.height + 1, r0 + rows))) return st;
    return SPCT_OK;
}

void put_u32(unsigned char* b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
}
uint32_t get_u32(const unsigned char* b) {
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}

// integral.cpp:636-650 header checks; the element size is checked by the caller.
spct_status read_header(FILE* f, const std::string& path, int* bins, int* h, int* w, int* elem) {
    unsigned char hdr[20];
    const size_t got = std::fread(hdr, 1, 20, f);
    if (got < 4 || std::memcmp(hdr, "IHT1", 4) != 0) return io("bad tensor magic: " + path);
    if (got < 20) return io("truncated tensor header: " + path);
    *bins = static_cast<int>(get_u32(hdr + 4));
    *h = static_cast<int>(get_u32(hdr + 8));
    *w = static_cast<int>(get_u32(hdr + 12));
    *elem = static_cast<int>(get_u32(hdr + 16));
    return SPCT_OK;
}

}  // namespace spct_iht1

using namespace spct_iht1;

extern "C" spct_status spct_cu_ih_dump(const spct_ih* t, const char* path, int elem_bytes, void* stream) {
    if (auto st = check_ih(t)) return st;
    if (!t->data || !path) return contract("dump_tensor: null tensor data or path");
    if (elem_bytes != 8 && elem_bytes != 4) return contract("dump_tensor: elem_bytes must be 8 or 4");
    const std::string p(path);
    FILE* f = std::fopen(path, "wb");
    if (!f) return io("cannot write tensor: " + p);  // integral.cpp:621
    unsigned char hdr[20];
    std::memcpy(hdr, "IHT1", 4);
    put_u32(hdr + 4, static_cast<uint32_t>(t->bins));
    put_u32(hdr + 8, static_cast<uint32_t>(t->height));
    put_u32(hdr + 12, static_cast<uint32_t>(t->width));
    put_u32(hdr + 16, static_cast<uint32_t>(elem_bytes));
    bool ok = std::fwrite(hdr, 1, 20, f) == 20;
    Staging sb;
    cudaStream_t s = as_stream(stream);
    spct_status st = sb.init(static_cast<size_t>(kChunkBytes + (t->width + 1) * 8));
    // chunk i: widen on the device into buffer i&1, copy to pinned i&1, record; the fwrite
    // of chunk i-1 overlaps the device work of chunk i
    int64_t pending_bytes = -1;
    int pending_buf = 0;
    auto flush = [&]() {
        if (pending_bytes < 0) return;
        cudaEventSynchronize(sb.ev[pending_buf]);
        ok = ok && std::fwrite(sb.host[pending_buf], 1, pending_bytes, f) == static_cast<size_t>(pending_bytes);
        pending_bytes = -1;
    };
    if (st == SPCT_OK)
        st = for_chunks(*t, elem_bytes, [&](int i, int k, int r0, int r1) -> spct_status {
            const int b = i & 1;
            const int64_t n = static_cast<int64_t>(r1 - r0) * (t->width + 1);
            if (elem_bytes == 8)
                widen_rows_kernel<uint64_t><<<grid_n(n), 256, 0, s>>>(*t, k, r0, r1, static_cast<uint64_t*>(sb.dev[b]));
            else
                widen_rows_kernel<uint32_t><<<grid_n(n), 256, 0, s>>>(*t, k, r0, r1, static_cast<uint32_t*>(sb.dev[b]));
            if (auto e = launch_status("widen_rows_kernel")) return e;
            if (pending_bytes >= 0 && pending_buf == b) flush();
            if (auto e = cuda_status(cudaMemcpyAsync(sb.host[b], sb.dev[b], n * elem_bytes, cudaMemcpyDeviceToHost, s),
                                     "IHT1 copy"))
                return e;
            cudaEventRecord(sb.ev[b], s);
            flush();  // the previous chunk's write overlaps this chunk's device work
            pending_bytes = n * elem_bytes;
            pending_buf = b;
            return SPCT_OK;
        });
    if (st == SPCT_OK) flush();
    ok = (std::fclose(f) == 0) && ok;
    if (st != SPCT_OK) return st;
    if (!ok) return io("write failed: " + p);  // integral.cpp:631
    return SPCT_OK;
}

extern "C" spct_status spct_cu_ih_load_header(const char* path, int* bins, int* height, int* width, int* elem_bytes) {
    if (!path || !bins || !height || !width || !elem_bytes) return contract("load_tensor: null argument");
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return io("cannot open tensor: " + p);  // integral.cpp:636
    spct_status st = read_header(f, p, bins, height, width, elem_bytes);
    std::fclose(f);
    if (st) return st;
    if (*elem_bytes != 8 && *elem_bytes != 4) return io("unsupported element size: " + p);  // :647
    if (*bins <= 0 || *height <= 0 || *width <= 0) return io("bad tensor dimensions: " + p);  // :648-649
    return SPCT_OK;
}

extern "C" spct_status spct_cu_ih_load(const char* path, const spct_ih* t, void* stream) {
    int bins, h, w, elem;
    if (auto st = spct_cu_ih_load_header(path, &bins, &h, &w, &elem)) return st;
    if (auto st = check_ih(t)) return st;
    if (!t->data) return contract("load_tensor: null tensor data");
    if (t->bins != bins || t->height != h || t->width != w)
        return contract("load_tensor: tensor descriptor does not match the file header");
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return io("cannot open tensor: " + p);
    std::fseek(f, 20, SEEK_SET);
    Staging sb;
    cudaStream_t s = as_stream(stream);
    unsigned* flags = nullptr;
    spct_status st = sb.init(static_cast<size_t>(kChunkBytes + (w + 1) * 8));
    if (st == SPCT_OK) st = cuda_status(cudaMalloc(&flags, sizeof(unsigned)), "IHT1 flags");
    if (st == SPCT_OK) st = cuda_status(cudaMemsetAsync(flags, 0, sizeof(unsigned), s), "IHT1 flags");
    if (st == SPCT_OK)
        st = for_chunks(*t, elem, [&](int i, int k, int r0, int r1) -> spct_status {
            const int b = i & 1;
            const int64_t n = static_cast<int64_t>(r1 - r0) * (w + 1);
            cudaEventSynchronize(sb.ev[b]);  // the H2D that last used buffer b is done
            if (std::fread(sb.host[b], 1, n * elem, f) != static_cast<size_t>(n * elem))
                return io("truncated tensor payload: " + p);  // integral.cpp:655
            if (auto e = cuda_status(cudaMemcpyAsync(sb.dev[b], sb.host[b], n * elem, cudaMemcpyHostToDevice, s),
                                     "IHT1 copy"))
                return e;
            if (elem == 8)
                narrow_rows_kernel<uint64_t><<<grid_n(n), 256, 0, s>>>(*t, k, r0, r1,
                                                                       static_cast<const uint64_t*>(sb.dev[b]), flags);
            else
                narrow_rows_kernel<uint32_t><<<grid_n(n), 256, 0, s>>>(*t, k, r0, r1,
                                                                       static_cast<const uint32_t*>(sb.dev[b]), flags);
            if (auto e = launch_status("narrow_rows_kernel")) return e;
            cudaEventRecord(sb.ev[b], s);
            return SPCT_OK;
        });
    std::fclose(f);
    unsigned hflags = 0;
    if (st == SPCT_OK) st = cuda_status(cudaMemcpyAsync(&hflags, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, s),
                                        "IHT1 flags");
    if (st == SPCT_OK) st = cuda_status(cudaStreamSynchronize(s), "IHT1 load");
    if (flags) cudaFree(flags);
    if (st) return st;
    if (hflags & 2u) return io("tensor value exceeds the uint32 device cell: " + p);
    if (hflags & 1u) return io("nonzero padding cell in tensor: " + p);
    return SPCT_OK;
}
