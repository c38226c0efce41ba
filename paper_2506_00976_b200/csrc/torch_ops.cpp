// PyTorch extension that loads the C ABI (libgridot_b200.so, a linked
// dependency resolved next to this library) and registers its device entry
// points as torch operators on CUDA tensors, launched on the current stream:
//
//   torch.ops.gridot_b200.version() -> str
//   torch.ops.gridot_b200.sumpool(Tensor fine, int[] dims, int kappa,
//                                 Tensor? stats) -> Tensor
//   torch.ops.gridot_b200.weighted_cost(Tensor mu, Tensor nu, Tensor mu_c,
//       Tensor nu_c, Tensor centre_cost, Tensor? cost_table, int max_sq,
//       int[] dims, int kappa, float p, int mode) -> Tensor
//
// `paper_2506_00976_b200._native` loads this extension with
// torch.ops.load_library before binding the remaining C entry points with
// ctypes (the same library handle).  No computation happens here: argument
// checks, output allocation from PyTorch's caching allocator, one C call.
#include <ATen/core/Tensor.h>
#include <ATen/ops/empty.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include <string>
#include <vector>

#include "../../include/gridot_b200.h"

namespace {

void check_f64_cuda(const at::Tensor &t, const char *name) {
    TORCH_CHECK(t.is_cuda(), name, " must be a CUDA tensor");
    TORCH_CHECK(t.scalar_type() == at::kDouble, name, " must be float64");
    TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
}

void check_rc(int rc, const char *what) {
    TORCH_CHECK(rc == GDT_OK, what, " failed with status ", rc, ": ", gdt_last_error());
}

std::string version() { return std::string(gdt_version()); }

at::Tensor sumpool(const at::Tensor &fine, std::vector<int64_t> dims, int64_t kappa,
                   const c10::optional<at::Tensor> &stats) {
    check_f64_cuda(fine, "fine");
    TORCH_CHECK(fine.dim() == 2, "fine must be [batch, cells]");
    TORCH_CHECK(kappa >= 1, "kappa must be >= 1");
    int64_t n = 1;
    for (int64_t d : dims) {
        TORCH_CHECK(d % kappa == 0, "dims must be multiples of kappa (pad first)");
        n *= d / kappa;
    }
    at::Tensor out = at::empty({fine.size(0), n}, fine.options());
    double *st = nullptr;
    if (stats.has_value()) {
        check_f64_cuda(*stats, "stats");
        TORCH_CHECK(stats->numel() == fine.size(0) * n * 3, "stats must hold [batch, n, 3]");
        st = stats->data_ptr<double>();
    }
    auto stream = c10::cuda::getCurrentCUDAStream(fine.device().index());
    check_rc(gdt_sumpool_stats_f64(fine.data_ptr<double>(), out.data_ptr<double>(), st,
                                   fine.size(0), (int)dims.size(), dims.data(), (int)kappa,
                                   stream.stream()),
             "gdt_sumpool_stats_f64");
    return out;
}

at::Tensor weighted_cost(const at::Tensor &mu, const at::Tensor &nu, const at::Tensor &mu_c,
                         const at::Tensor &nu_c, const at::Tensor &centre_cost,
                         const c10::optional<at::Tensor> &cost_table, int64_t max_sq,
                         std::vector<int64_t> dims, int64_t kappa, double p, int64_t mode) {
    for (auto *t : {&mu, &nu, &mu_c, &nu_c, &centre_cost}) check_f64_cuda(*t, "operand");
    const int64_t B = mu.size(0), n = mu_c.size(1);
    at::Tensor out = at::empty({B, n, n}, mu.options());
    const double *tab = nullptr;
    if (cost_table.has_value()) {
        check_f64_cuda(*cost_table, "cost_table");
        tab = cost_table->data_ptr<double>();
    }
    auto stream = c10::cuda::getCurrentCUDAStream(mu.device().index());
    check_rc(gdt_weighted_cost(mu.data_ptr<double>(), nu.data_ptr<double>(),
                               mu_c.data_ptr<double>(), nu_c.data_ptr<double>(),
                               centre_cost.data_ptr<double>(), tab, max_sq,
                               out.data_ptr<double>(), nullptr, B, (int)dims.size(), dims.data(),
                               (int)kappa, p, (int)mode, stream.stream()),
             "gdt_weighted_cost");
    return out;
}

}  // namespace

TORCH_LIBRARY(gridot_b200, m) {
    m.def("version() -> str", &version);
    m.def("sumpool(Tensor fine, int[] dims, int kappa, Tensor? stats) -> Tensor");
    m.def("weighted_cost(Tensor mu, Tensor nu, Tensor mu_c, Tensor nu_c, Tensor centre_cost, "
          "Tensor? cost_table, int max_sq, int[] dims, int kappa, float p, int mode) -> Tensor");
}

TORCH_LIBRARY_IMPL(gridot_b200, CUDA, m) {
    m.impl("sumpool", &sumpool);
    m.impl("weighted_cost", &weighted_cost);
}
