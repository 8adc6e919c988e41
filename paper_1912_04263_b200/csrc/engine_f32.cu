// engine_f32.cu — the float engine: explicit instantiation of Workspace<float> and
// Sharded<float> plus the typed entry points behind IEngine (workspace.cuh).
// engine.cu, engine_f64.cu and engine_f32.cu compile in parallel (build.py).
#include "workspace.cuh"
#include "shard.cuh"

namespace qpcg_b200 {

template class Workspace<float>;
template class Sharded<float>;

template <>
IEngine<float>* make_engine<float>(bool sharded) {
  if (sharded) return new Sharded<float>();
  return new Workspace<float>();
}

template <>
void validate_settings_in<float>(const qpcg_settings& s) {
  Workspace<float>::validate_settings(s);
}

// y = M x through the plan-driven SpMV (operator-level entry point)
template <>
void op_spmv<float>(const HostCsr<float>& mv, const float* x, float* y, int device) {
  using T = float;
  if (device >= 0) CK(cudaSetDevice(device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  AllocScope scope(s);
  CubTemp tmp;
  DevCsr<T> M{mv.rows, mv.cols, mv.nnz, nullptr, nullptr, nullptr};
  T *dx, *dy;
  CK(dmalloc(&M.val, sizeof(T) * (M.nnz + 1)));
  CK(dmalloc(&M.ci, 4 * (size_t(M.nnz) + 1)));
  CK(dmalloc(&M.rp, 4 * (size_t(M.rows) + 1)));
  CK(dmalloc(&dx, sizeof(T) * (M.cols + 1)));
  CK(dmalloc(&dy, sizeof(T) * (M.rows + 1)));
  CK(cudaMemcpyAsync(M.val, mv.values, sizeof(T) * M.nnz, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(M.ci, mv.col_indices, 4 * size_t(M.nnz), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(M.rp, mv.row_ptr, 4 * (size_t(M.rows) + 1), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dx, x, sizeof(T) * M.cols, cudaMemcpyHostToDevice, s));
  SpmvPlan<T> P = plan_build<T>(M.rp, M.rows, M.nnz, tmp, s);
  if (Workspace<T>::compress_indices()) plan_compress(P, M.ci, M.nnz, M.cols, tmp, s);  // as the workspace
  launch_spmv<T, 1, SumOp>(M, P, GatherVec<T>{dx}, EpiStore<T>{dy}, s);
  CK(cudaMemcpyAsync(y, dy, sizeof(T) * M.rows, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  plan_free(P);
  dfree(M.val);
  dfree(M.ci);
  dfree(M.rp);
  dfree(dx);
  dfree(dy);
  if (tmp.ptr) dfree(tmp.ptr);
  tmp.ptr = nullptr;
  CK(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
}

template <>
void op_pcg<float>(const HostCsr<float>& pf, const HostCsr<float>& a, const HostCsr<float>& at, float sigma,
                float rho, const float* b, const float* warm, float eps, uint32_t max_iter, float* x,
                double* res, int device) {
  Workspace<float> w;
  w.setup_operator(pf, a, at, sigma, rho, device);
  w.op_pcg(b, warm, eps, max_iter, x, res);
}

}  // namespace qpcg_b200
