// Fused build + match entry point (placeholder schedule: build, then match on the
// freshly written slab).  The single-pass kernel replaces this in DESIGN.md §4.
#include "spct_internal.h"

using namespace spct_impl;

extern "C" spct_status spct_cu_ih_build_match(const spct_source* src, const spct_ih* out, const double* tmpl, int kw,
                                              int kh, double p, int metric, double* partial, void* workspace,
                                              size_t workspace_bytes, void* stream) {
    if (!out || !out->data) return contract("ih_build_match: this schedule needs tensor storage");
    if (auto st = spct_cu_ih_build(src, out, workspace, workspace_bytes, stream)) return st;
    return spct_cu_hist_partial(out, tmpl, kw, kh, p, metric, partial, 0, stream);
}
