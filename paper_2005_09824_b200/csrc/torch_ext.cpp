// PyTorch C++ extension: tensor/stream plumbing over the C-ABI in lfmmi.h.
// No compute here — every entry point validates tensors, picks up the current
// CUDA stream and forwards plain pointers to libpaper_lfmmi.so.
#include <torch/extension.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>

#include <cstdint>
#include <string>

#include "lfmmi.h"

namespace {

void check(int rc, const char *what) {
  if (rc != LFMMI_OK) {
    const std::string msg = std::string(what) + ": " + lfmmi_last_error();
    if (rc == LFMMI_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
}

void need_cpu(const torch::Tensor &t, torch::ScalarType dt, const char *name) {
  TORCH_CHECK(t.device().is_cpu(), name, " must be a CPU tensor");
  TORCH_CHECK(t.scalar_type() == dt, name, " has the wrong dtype");
  TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
}

void need_cuda(const torch::Tensor &t, torch::ScalarType dt, const char *name) {
  TORCH_CHECK(t.is_cuda(), name, " must be a CUDA tensor");
  TORCH_CHECK(t.scalar_type() == dt, name, " has the wrong dtype");
  TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
}

template <typename T>
T *ptr_or_null(const c10::optional<torch::Tensor> &t) {
  return t.has_value() && t->defined() ? static_cast<T *>(t->data_ptr()) : nullptr;
}

lfmmi_graphs *as_graphs(int64_t h) { return reinterpret_cast<lfmmi_graphs *>(h); }

int precision_of(const torch::Tensor &t) {
  if (t.scalar_type() == torch::kFloat32) return LFMMI_F32;
  TORCH_CHECK(t.scalar_type() == torch::kFloat64, "real tensors must be float32 or float64");
  return LFMMI_F64;
}

void *stream_of(const torch::Tensor &t) {
  return static_cast<void *>(at::cuda::getCurrentCUDAStream(t.device().index()).stream());
}

}  // namespace

int64_t graphs_create(int64_t num_pdfs, torch::Tensor row_num_states, torch::Tensor row_num_arcs,
                      torch::Tensor fw_from, torch::Tensor fw_to, torch::Tensor fw_pdf,
                      torch::Tensor fw_prob, c10::optional<torch::Tensor> bw_from,
                      c10::optional<torch::Tensor> bw_to, c10::optional<torch::Tensor> bw_pdf,
                      c10::optional<torch::Tensor> bw_prob, torch::Tensor final_probs,
                      torch::Tensor initial_states) {
  need_cpu(row_num_states, torch::kInt64, "row_num_states");
  need_cpu(row_num_arcs, torch::kInt64, "row_num_arcs");
  need_cpu(fw_from, torch::kInt32, "fw_from");
  need_cpu(fw_to, torch::kInt32, "fw_to");
  need_cpu(fw_pdf, torch::kInt32, "fw_pdf");
  need_cpu(fw_prob, torch::kFloat64, "fw_prob");
  need_cpu(final_probs, torch::kFloat64, "final_probs");
  need_cpu(initial_states, torch::kInt32, "initial_states");
  TORCH_CHECK(fw_from.dim() == 2 && final_probs.dim() == 2, "padded (G, I) / (G, S) layouts expected");
  const bool bw = bw_from.has_value() && bw_from->defined();
  if (bw) {
    need_cpu(*bw_from, torch::kInt32, "bw_from");
    need_cpu(*bw_to, torch::kInt32, "bw_to");
    need_cpu(*bw_pdf, torch::kInt32, "bw_pdf");
    need_cpu(*bw_prob, torch::kFloat64, "bw_prob");
  }
  lfmmi_graphs *g = nullptr;
  // uint32 index arrays are passed as int32 bit patterns (values < 2^31).
  check(lfmmi_graphs_create(
            int32_t(fw_from.size(0)), int32_t(final_probs.size(1)), int32_t(fw_from.size(1)),
            int32_t(num_pdfs), row_num_states.data_ptr<int64_t>(), row_num_arcs.data_ptr<int64_t>(),
            reinterpret_cast<const uint32_t *>(fw_from.data_ptr<int32_t>()),
            reinterpret_cast<const uint32_t *>(fw_to.data_ptr<int32_t>()),
            reinterpret_cast<const uint32_t *>(fw_pdf.data_ptr<int32_t>()),
            fw_prob.data_ptr<double>(),
            bw ? reinterpret_cast<const uint32_t *>(bw_from->data_ptr<int32_t>()) : nullptr,
            bw ? reinterpret_cast<const uint32_t *>(bw_to->data_ptr<int32_t>()) : nullptr,
            bw ? reinterpret_cast<const uint32_t *>(bw_pdf->data_ptr<int32_t>()) : nullptr,
            bw ? bw_prob->data_ptr<double>() : nullptr, final_probs.data_ptr<double>(),
            reinterpret_cast<const uint32_t *>(initial_states.data_ptr<int32_t>()), &g),
        "lfmmi_graphs_create");
  return reinterpret_cast<int64_t>(g);
}

// Linear-chain batch over caller-owned device tensors (lfmmi_graphs_create_linear):
// `items` (rows, 4) int32, `states` (sum S, 4) int32 (bit patterns).  The
// Python owner keeps both tensors alive as long as the handle.
int64_t graphs_create_linear(int64_t max_states, int64_t num_pdfs, torch::Tensor items,
                             torch::Tensor states) {
  need_cuda(items, torch::kInt32, "items");
  need_cuda(states, torch::kInt32, "states");
  TORCH_CHECK(items.dim() == 2 && items.size(1) == 4, "items must be (rows, 4)");
  TORCH_CHECK(states.dim() == 2 && states.size(1) == 4, "states must be (sum S, 4)");
  lfmmi_graphs *g = nullptr;
  check(lfmmi_graphs_create_linear(int32_t(items.size(0)), int32_t(max_states), int32_t(num_pdfs),
                                   items.data_ptr<int32_t>(),
                                   reinterpret_cast<const uint32_t *>(states.data_ptr<int32_t>()), &g),
        "lfmmi_graphs_create_linear");
  return reinterpret_cast<int64_t>(g);
}

void set_option(const std::string &name, const std::string &value) {
  check(lfmmi_set_option(name.c_str(), value.c_str()), "lfmmi_set_option");
}

std::string get_option(const std::string &name) {
  char buf[256];
  check(lfmmi_get_option(name.c_str(), buf, sizeof(buf)), "lfmmi_get_option");
  return buf;
}

void reset_options() { lfmmi_reset_options(); }

void graphs_destroy(int64_t h) { check(lfmmi_graphs_destroy(as_graphs(h)), "lfmmi_graphs_destroy"); }

int64_t workspace_size(int64_t max_states, int64_t total_frames, int64_t precision) {
  return int64_t(lfmmi_workspace_size(int32_t(max_states), total_frames, int32_t(precision)));
}

// Every per-item array must hold exactly B entries: a numerator list or a
// lengths vector of the wrong size would otherwise index past its end on the
// device.  (Lengths outside [1, T_max] are caught on the device: item_frames.)
void check_batch_sizes(int64_t B, const torch::Tensor &lengths,
                       std::initializer_list<const torch::Tensor *> per_item) {
  TORCH_CHECK(lengths.dim() == 1 && lengths.numel() == B, "lengths must have ", B,
              " entries, got ", lengths.numel());
  for (const torch::Tensor *t : per_item)
    TORCH_CHECK(t->numel() == B, "per-item array has ", t->numel(), " entries, batch has ", B);
}

int64_t chain_loss_workspace_size(int64_t num_h, int64_t den_h, int64_t batch, int64_t max_frames,
                                  int64_t num_pdfs, int64_t total_frames, int64_t precision) {
  return int64_t(lfmmi_chain_loss_workspace_size(
      as_graphs(num_h), as_graphs(den_h), int32_t(batch), int32_t(max_frames), int32_t(num_pdfs),
      total_frames, int32_t(precision)));
}

void forward_backward(int64_t h, torch::Tensor row_map, torch::Tensor loglikes,
                      torch::Tensor lengths, double leak, double scale_floor,
                      c10::optional<torch::Tensor> leak_pi, int64_t total_frames,
                      torch::Tensor workspace,
                      torch::Tensor posteriors, int64_t post_mode,
                      c10::optional<torch::Tensor> other_fail, torch::Tensor log_probs,
                      torch::Tensor fail_frames, c10::optional<torch::Tensor> scale_logs) {
  const c10::cuda::CUDAGuard guard(loglikes.device());
  const auto dt = loglikes.scalar_type();
  need_cuda(row_map, torch::kInt64, "row_map");
  need_cuda(loglikes, dt, "loglikes");
  need_cuda(lengths, torch::kInt32, "lengths");
  need_cuda(workspace, torch::kUInt8, "workspace");
  need_cuda(posteriors, dt, "posteriors");
  need_cuda(log_probs, torch::kFloat64, "log_probs");
  need_cuda(fail_frames, torch::kInt32, "fail_frames");
  if (leak_pi.has_value() && leak_pi->defined()) need_cuda(*leak_pi, dt, "leak_pi");
  TORCH_CHECK(loglikes.dim() == 3, "loglikes must be (B, T, D)");
  check_batch_sizes(loglikes.size(0), lengths, {&row_map});
  TORCH_CHECK(posteriors.sizes() == loglikes.sizes(), "posteriors must match loglikes");
  TORCH_CHECK(log_probs.numel() == loglikes.size(0) && fail_frames.numel() == loglikes.size(0),
              "log_probs / fail_frames must have B entries");
  check(lfmmi_forward_backward(as_graphs(h), row_map.data_ptr<int64_t>(), int32_t(loglikes.size(0)),
                               int32_t(loglikes.size(1)), int32_t(loglikes.size(2)),
                               precision_of(loglikes), loglikes.data_ptr(),
                               lengths.data_ptr<int32_t>(), leak, scale_floor,
                               ptr_or_null<void>(leak_pi), total_frames, workspace.data_ptr(),
                               size_t(workspace.numel()), posteriors.data_ptr(), int32_t(post_mode),
                               ptr_or_null<int32_t>(other_fail), log_probs.data_ptr<double>(),
                               fail_frames.data_ptr<int32_t>(), ptr_or_null<double>(scale_logs),
                               stream_of(loglikes)),
        "lfmmi_forward_backward");
}

void chain_loss(int64_t num_h, torch::Tensor num_row_map, int64_t den_h, torch::Tensor den_row_map,
                torch::Tensor loglikes, torch::Tensor lengths, double leak, double scale_floor,
                c10::optional<torch::Tensor> num_leak_pi, c10::optional<torch::Tensor> den_leak_pi,
                int64_t total_frames, torch::Tensor workspace, torch::Tensor grad, torch::Tensor num_log_probs,
                torch::Tensor den_log_probs, torch::Tensor num_fail, torch::Tensor den_fail,
                torch::Tensor totals) {
  const c10::cuda::CUDAGuard guard(loglikes.device());
  const auto dt = loglikes.scalar_type();
  need_cuda(num_row_map, torch::kInt64, "num_row_map");
  need_cuda(den_row_map, torch::kInt64, "den_row_map");
  need_cuda(loglikes, dt, "loglikes");
  need_cuda(lengths, torch::kInt32, "lengths");
  need_cuda(workspace, torch::kUInt8, "workspace");
  need_cuda(grad, dt, "grad");
  need_cuda(num_log_probs, torch::kFloat64, "num_log_probs");
  need_cuda(den_log_probs, torch::kFloat64, "den_log_probs");
  need_cuda(num_fail, torch::kInt32, "num_fail");
  need_cuda(den_fail, torch::kInt32, "den_fail");
  need_cuda(totals, torch::kFloat64, "totals");
  TORCH_CHECK(loglikes.dim() == 3, "loglikes must be (B, T, D)");
  TORCH_CHECK(grad.sizes() == loglikes.sizes(), "grad must match loglikes");
  check_batch_sizes(loglikes.size(0), lengths, {&num_row_map, &den_row_map, &num_log_probs,
                                                &den_log_probs, &num_fail, &den_fail});
  TORCH_CHECK(totals.numel() >= 3, "totals must hold 3 doubles");
  check(lfmmi_chain_loss(as_graphs(num_h), num_row_map.data_ptr<int64_t>(), as_graphs(den_h),
                         den_row_map.data_ptr<int64_t>(), int32_t(loglikes.size(0)),
                         int32_t(loglikes.size(1)), int32_t(loglikes.size(2)),
                         precision_of(loglikes), loglikes.data_ptr(), lengths.data_ptr<int32_t>(),
                         leak, scale_floor, ptr_or_null<void>(num_leak_pi),
                         ptr_or_null<void>(den_leak_pi), total_frames, workspace.data_ptr(),
                         size_t(workspace.numel()), grad.data_ptr(),
                         num_log_probs.data_ptr<double>(), den_log_probs.data_ptr<double>(),
                         num_fail.data_ptr<int32_t>(), den_fail.data_ptr<int32_t>(),
                         totals.data_ptr<double>(), stream_of(loglikes)),
        "lfmmi_chain_loss");
}

// Ragged input: loglikes (sum_b T_b, D), item b at rows [sum_{j<b} T_j, ...).
void chain_loss_packed(int64_t num_h, torch::Tensor num_row_map, int64_t den_h,
                       torch::Tensor den_row_map, torch::Tensor loglikes, torch::Tensor lengths,
                       int64_t max_frames, double leak, double scale_floor, int64_t total_frames,
                       torch::Tensor workspace, torch::Tensor grad, torch::Tensor num_log_probs,
                       torch::Tensor den_log_probs, torch::Tensor num_fail, torch::Tensor den_fail,
                       torch::Tensor totals) {
  const c10::cuda::CUDAGuard guard(loglikes.device());
  const auto dt = loglikes.scalar_type();
  need_cuda(num_row_map, torch::kInt64, "num_row_map");
  need_cuda(den_row_map, torch::kInt64, "den_row_map");
  need_cuda(loglikes, dt, "loglikes");
  need_cuda(lengths, torch::kInt32, "lengths");
  need_cuda(workspace, torch::kUInt8, "workspace");
  need_cuda(grad, dt, "grad");
  need_cuda(totals, torch::kFloat64, "totals");
  TORCH_CHECK(loglikes.dim() == 2, "packed loglikes must be (sum T, D)");
  TORCH_CHECK(grad.sizes() == loglikes.sizes(), "grad must match loglikes");
  need_cuda(num_log_probs, torch::kFloat64, "num_log_probs");
  need_cuda(den_log_probs, torch::kFloat64, "den_log_probs");
  need_cuda(num_fail, torch::kInt32, "num_fail");
  need_cuda(den_fail, torch::kInt32, "den_fail");
  check_batch_sizes(lengths.size(0), lengths, {&num_row_map, &den_row_map, &num_log_probs,
                                               &den_log_probs, &num_fail, &den_fail});
  TORCH_CHECK(totals.numel() >= 3, "totals must hold 3 doubles");
  TORCH_CHECK(total_frames == loglikes.size(0), "total_frames must equal the packed row count");
  check(lfmmi_chain_loss_packed(
            as_graphs(num_h), num_row_map.data_ptr<int64_t>(), as_graphs(den_h),
            den_row_map.data_ptr<int64_t>(), int32_t(lengths.size(0)), int32_t(max_frames),
            int32_t(loglikes.size(1)), precision_of(loglikes), loglikes.data_ptr(),
            lengths.data_ptr<int32_t>(), leak, scale_floor, nullptr, nullptr, total_frames,
            workspace.data_ptr(), size_t(workspace.numel()), grad.data_ptr(),
            num_log_probs.data_ptr<double>(), den_log_probs.data_ptr<double>(),
            num_fail.data_ptr<int32_t>(), den_fail.data_ptr<int32_t>(), totals.data_ptr<double>(),
            stream_of(loglikes)),
        "lfmmi_chain_loss_packed");
}

void forward_kernel(int64_t h, torch::Tensor row_map, torch::Tensor expl, torch::Tensor lengths,
                    double leak, torch::Tensor leak_pi, double scale_floor, torch::Tensor alpha,
                    torch::Tensor scales, torch::Tensor fail_frames) {
  const c10::cuda::CUDAGuard guard(expl.device());
  need_cuda(row_map, torch::kInt64, "row_map");
  need_cuda(expl, torch::kFloat64, "expl");
  need_cuda(lengths, torch::kInt32, "lengths");
  need_cuda(leak_pi, torch::kFloat64, "leak_pi");
  need_cuda(alpha, torch::kFloat64, "alpha");
  need_cuda(scales, torch::kFloat64, "scales");
  need_cuda(fail_frames, torch::kInt64, "fail_frames");
  check(lfmmi_forward_kernel(as_graphs(h), row_map.data_ptr<int64_t>(), int32_t(expl.size(0)),
                             int32_t(expl.size(1)), int32_t(expl.size(2)), expl.data_ptr<double>(),
                             lengths.data_ptr<int32_t>(), leak, leak_pi.data_ptr<double>(),
                             scale_floor, alpha.data_ptr<double>(), scales.data_ptr<double>(),
                             fail_frames.data_ptr<int64_t>(), stream_of(expl)),
        "lfmmi_forward_kernel");
}

void backward_kernel(int64_t h, torch::Tensor row_map, torch::Tensor expl, torch::Tensor lengths,
                     torch::Tensor scales, double leak, torch::Tensor leak_pi,
                     torch::Tensor fail_frames, torch::Tensor beta) {
  const c10::cuda::CUDAGuard guard(expl.device());
  need_cuda(row_map, torch::kInt64, "row_map");
  need_cuda(expl, torch::kFloat64, "expl");
  need_cuda(lengths, torch::kInt32, "lengths");
  need_cuda(scales, torch::kFloat64, "scales");
  need_cuda(leak_pi, torch::kFloat64, "leak_pi");
  need_cuda(fail_frames, torch::kInt64, "fail_frames");
  need_cuda(beta, torch::kFloat64, "beta");
  check(lfmmi_backward_kernel(as_graphs(h), row_map.data_ptr<int64_t>(), int32_t(expl.size(0)),
                              int32_t(expl.size(1)), int32_t(expl.size(2)), expl.data_ptr<double>(),
                              lengths.data_ptr<int32_t>(), scales.data_ptr<double>(), leak,
                              leak_pi.data_ptr<double>(), fail_frames.data_ptr<int64_t>(),
                              beta.data_ptr<double>(), stream_of(expl)),
        "lfmmi_backward_kernel");
}

void posterior_kernel(int64_t h, torch::Tensor row_map, torch::Tensor expl, torch::Tensor lengths,
                      torch::Tensor alpha, torch::Tensor beta, torch::Tensor fail_frames,
                      torch::Tensor gamma) {
  const c10::cuda::CUDAGuard guard(expl.device());
  need_cuda(row_map, torch::kInt64, "row_map");
  need_cuda(expl, torch::kFloat64, "expl");
  need_cuda(lengths, torch::kInt32, "lengths");
  need_cuda(alpha, torch::kFloat64, "alpha");
  need_cuda(beta, torch::kFloat64, "beta");
  need_cuda(fail_frames, torch::kInt64, "fail_frames");
  need_cuda(gamma, torch::kFloat64, "gamma");
  check(lfmmi_posterior_kernel(as_graphs(h), row_map.data_ptr<int64_t>(), int32_t(expl.size(0)),
                               int32_t(expl.size(1)), int32_t(expl.size(2)),
                               expl.data_ptr<double>(), lengths.data_ptr<int32_t>(),
                               alpha.data_ptr<double>(), beta.data_ptr<double>(),
                               fail_frames.data_ptr<int64_t>(), gamma.data_ptr<double>(),
                               stream_of(expl)),
        "lfmmi_posterior_kernel");
}

std::string version() { return lfmmi_version(); }
int64_t last_launch_count() { return lfmmi_last_launch_count(); }
std::string last_den_kernel() { return lfmmi_last_den_kernel(); }
std::string last_kernel() { return lfmmi_last_kernel(); }

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
  m.def("graphs_create", &graphs_create);
  m.def("graphs_destroy", &graphs_destroy);
  m.def("graphs_create_linear", &graphs_create_linear);
  m.def("set_option", &set_option);
  m.def("get_option", &get_option);
  m.def("reset_options", &reset_options);
  m.def("workspace_size", &workspace_size);
  m.def("chain_loss_workspace_size", &chain_loss_workspace_size);
  m.def("forward_backward", &forward_backward);
  m.def("chain_loss", &chain_loss);
  m.def("chain_loss_packed", &chain_loss_packed);
  m.def("forward_kernel", &forward_kernel);
  m.def("backward_kernel", &backward_kernel);
  m.def("posterior_kernel", &posterior_kernel);
  m.def("version", &version);
  m.def("last_launch_count", &last_launch_count);
  m.def("last_den_kernel", &last_den_kernel);
  m.def("last_kernel", &last_kernel);
}
