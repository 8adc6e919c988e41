// Minimal repro for the compute-sanitizer synccheck report on kernels inside
// a CUDA-graph conditional (WHILE) node body (profiles/r02_synccheck_repro.txt).
//
// One trivial kernel: every thread of a full warp does one __shfl_xor_sync
// with the full mask and one __syncthreads (no divergence is possible).  It is
// run three ways:
//   plain   - launched from the host
//   graph   - as a kernel node of an ordinary CUDA graph
//   while   - as a kernel node of the body graph of a WHILE conditional node
//             (the body also holds a one-thread kernel that counts down and
//             clears the condition after 3 iterations)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/synccheck_cond synccheck_cond.cu
//   compute-sanitizer --tool synccheck /tmp/synccheck_cond plain|graph|while [blocks]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      std::printf("%s failed: %s\n", #x, cudaGetErrorString(e));                  \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

__global__ void k_shfl(float* out) {
  float v = float(threadIdx.x);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

__global__ void k_count(int* counter, cudaGraphConditionalHandle h) {
  const int left = --(*counter);
  cudaGraphSetConditional(h, left > 0 ? 1u : 0u);
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "while";
  const unsigned blocks = argc > 2 ? unsigned(std::atoi(argv[2])) : 3u;  // grid of k_shfl
  float* out;
  int* counter;
  CK(cudaMalloc(&out, sizeof(float) * 256 * blocks));
  CK(cudaMalloc(&counter, sizeof(int)));
  const int three = 3;
  CK(cudaMemcpy(counter, &three, sizeof(int), cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  if (!std::strcmp(mode, "plain")) {
    k_shfl<<<blocks, 256, 0, s>>>(out);
    CK(cudaGetLastError());
  } else {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraph_t body = g;
    cudaGraphConditionalHandle h{};
    if (!std::strcmp(mode, "while")) {
      CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cn;
      CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
      body = cp.conditional.phGraph_out[0];
    }
    cudaGraphNode_t n1;
    cudaKernelNodeParams kp = {};
    void* a1[] = {&out};
    kp.func = (void*)k_shfl;
    kp.gridDim = dim3(blocks);
    kp.blockDim = dim3(256);
    kp.kernelParams = a1;
    CK(cudaGraphAddKernelNode(&n1, body, nullptr, 0, &kp));
    if (!std::strcmp(mode, "while")) {
      cudaGraphNode_t n2;
      void* a2[] = {&counter, &h};
      kp.func = (void*)k_count;
      kp.gridDim = dim3(1);
      kp.blockDim = dim3(1);
      kp.kernelParams = a2;
      CK(cudaGraphAddKernelNode(&n2, body, &n1, 1, &kp));
    }
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
  }
  CK(cudaStreamSynchronize(s));
  float h[4];
  CK(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
  int left = -1;
  CK(cudaMemcpy(&left, counter, sizeof(int), cudaMemcpyDeviceToHost));
  std::printf("%s: out[0..3] = %g %g %g %g, counter %d (expect 1 1 5 5; 0 for while)\n", mode,
              h[0], h[1], h[2], h[3], left);
  return 0;
}
