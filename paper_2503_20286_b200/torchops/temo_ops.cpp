// TORCH_LIBRARY registration of the C ABI: torch.ops.temo.* call the same entry
// points as the ctypes binding, on the current CUDA stream, with torch-allocated outputs and
// workspace -- so they can be captured in CUDA graphs and traced by torch.compile (Meta
// kernels give the output shapes).  No arithmetic here: every op is one or two C-ABI calls.
#include <torch/library.h>
#include <ATen/ATen.h>
#include <c10/cuda/CUDAStream.h>
#include <c10/cuda/CUDAGuard.h>

#include <cstring>
#include <vector>

#include "temo_b200.h"

namespace {

void check_rc(int rc, const char *what) {
    TORCH_CHECK(rc == TEMO_OK, "temo::", what, " failed with status ", rc);
}

at::Tensor f64_2d(const at::Tensor &t, const char *name) {
    TORCH_CHECK(t.is_cuda() && t.dim() == 2 && t.scalar_type() == at::kDouble, name,
                " must be a 2-D float64 CUDA tensor");
    return t.contiguous();
}

temo_stream_t stream_of(const at::Tensor &t) {
    return (temo_stream_t)c10::cuda::getCurrentCUDAStream(t.device().index()).stream();
}

// ndsort.rank_assign (ndsort.py:47-71): ranks, l, number of fronts, status word
std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor> rank_cuda(const at::Tensor &F_, int64_t n,
                                                                     int64_t mode) {
    const at::Tensor F = f64_2d(F_, "F");
    c10::cuda::CUDAGuard g(F.device());
    const int64_t N = F.size(0);
    const int m = (int)F.size(1);
    auto i32 = F.options().dtype(at::kInt);
    at::Tensor rank = at::empty({N}, i32), l = at::empty({1}, i32), nf = at::empty({1}, i32);
    at::Tensor status = at::zeros({1}, i32);
    const size_t wsb = temo_rank_ws_bytes(N, m);
    at::Tensor ws = at::empty({(int64_t)(wsb > 0 ? wsb : 1)}, F.options().dtype(at::kByte));
    check_rc(temo_rank(F.data_ptr<double>(), N, m, n, (int)mode, rank.data_ptr<int32_t>(), l.data_ptr<int32_t>(),
                       nf.data_ptr<int32_t>(), status.data_ptr<int32_t>(), ws.data_ptr(), wsb, stream_of(F)),
             "rank");
    return {rank, l, nf, status};
}

std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor> rank_meta(const at::Tensor &F, int64_t, int64_t) {
    auto i32 = F.options().dtype(at::kInt);
    return {at::empty({F.size(0)}, i32), at::empty({1}, i32), at::empty({1}, i32), at::empty({1}, i32)};
}

// problems.evaluate (problems.py:105-136; LSMOP1-9): problem id, objective count, LSMOP groups
at::Tensor evaluate_cuda(const at::Tensor &X_, int64_t problem_id, int64_t m, int64_t nk, at::IntArrayRef sublen,
                         at::IntArrayRef offset) {
    const at::Tensor X = f64_2d(X_, "X");
    c10::cuda::CUDAGuard g(X.device());
    temo_problem p;
    std::memset(&p, 0, sizeof(p));
    p.id = (int32_t)problem_id;
    p.m = (int32_t)m;
    p.d = X.size(1);
    p.nk = (int32_t)nk;
    TORCH_CHECK(sublen.size() <= 16 && offset.size() <= 17, "at most 16 objectives");
    for (size_t i = 0; i < sublen.size(); ++i) p.sublen[i] = (int32_t)sublen[i];
    for (size_t i = 0; i < offset.size(); ++i) p.offset[i] = (int32_t)offset[i];
    at::Tensor F = at::empty({X.size(0), m}, X.options());
    check_rc(temo_evaluate(&p, X.data_ptr<double>(), X.size(0), F.data_ptr<double>(), stream_of(X)), "evaluate");
    return F;
}

at::Tensor evaluate_meta(const at::Tensor &X, int64_t, int64_t m, int64_t, at::IntArrayRef, at::IntArrayRef) {
    return at::empty({X.size(0), m}, X.options());
}

// indicators.igd (indicators.py:19-26)
at::Tensor igd_cuda(const at::Tensor &F_, const at::Tensor &R_) {
    const at::Tensor F = f64_2d(F_, "F"), R = f64_2d(R_, "Fstar");
    TORCH_CHECK(F.size(1) == R.size(1), "F and Fstar need the same objective count");
    c10::cuda::CUDAGuard g(F.device());
    at::Tensor out = at::empty({1}, F.options());
    const size_t wsb = temo_igd_ws_bytes(R.size(0));
    at::Tensor ws = at::empty({(int64_t)(wsb > 0 ? wsb : 1)}, F.options().dtype(at::kByte));
    check_rc(temo_igd(F.data_ptr<double>(), F.size(0), (int)F.size(1), R.data_ptr<double>(), R.size(0),
                      out.data_ptr<double>(), ws.data_ptr(), wsb, stream_of(F)),
             "igd");
    return out;
}

at::Tensor igd_meta(const at::Tensor &F, const at::Tensor &) { return at::empty({1}, F.options()); }

}  // namespace

TORCH_LIBRARY(temo, m) {
    m.def("rank(Tensor F, int n, int mode) -> (Tensor rank, Tensor l, Tensor nfronts, Tensor status)");
    m.def("evaluate(Tensor X, int problem_id, int m, int nk, int[] sublen, int[] offset) -> Tensor");
    m.def("igd(Tensor F, Tensor Fstar) -> Tensor");
}

TORCH_LIBRARY_IMPL(temo, CUDA, m) {
    m.impl("rank", rank_cuda);
    m.impl("evaluate", evaluate_cuda);
    m.impl("igd", igd_cuda);
}

TORCH_LIBRARY_IMPL(temo, Meta, m) {
    m.impl("rank", rank_meta);
    m.impl("evaluate", evaluate_meta);
    m.impl("igd", igd_meta);
}
