// Can the reference's N(0,1) draws be produced on the device bit for bit?
// (§8(f) rank 2, GPU instance generation.)
//
// The reference draws normal = sqrt(-2 log u1) * cos(2 pi u2) with u1, u2 from
// its counter-based splitmix64 stream (bench/rng.hpp:39-88; restated in
// paper_1912_04263_b200/csrc/gen.cpp:36-70) through glibc's log and cos.  This
// program evaluates the same expression for N draws on the host (glibc, the
// same libm the reference links) and on the device (CUDA's double-precision
// log / cos; sqrt and the products are IEEE-exact on both sides: -ffp-contract=off
// and --fmad=false) and counts the draws whose bits differ, per function.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -Xcompiler -ffp-contract=off \
//        -O3 -o /tmp/gen_normals_device gen_normals_device.cu
//   /tmp/gen_normals_device [N = 100000000]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

using u64 = uint64_t;
constexpr u64 kGolden = 0x9E3779B97F4A7C15ULL;
constexpr double kPi = 3.141592653589793238462643383279502884;

__host__ __device__ inline u64 mix64(u64 z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
__host__ __device__ inline double u01_at(u64 key, u64 pos) {
  return static_cast<double>(mix64(key + pos * kGolden) >> 11) * 0x1.0p-53;
}

__global__ void k_draws(u64 key, u64 n, double* lg, double* cs, double* nv) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const double u1 = 1.0 - u01_at(key, 2 * i);
    const double u2 = u01_at(key, 2 * i + 1);
    const double l = log(u1), c = cos(2.0 * kPi * u2);
    lg[i] = l;
    cs[i] = c;
    nv[i] = sqrt(-2.0 * l) * c;
  }
}

static u64 bits(double d) {
  u64 b;
  std::memcpy(&b, &d, 8);
  return b;
}

int main(int argc, char** argv) {
  const u64 n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000000ull;
  const u64 key = mix64(0x5eed ^ kGolden);  // any stream key
  const u64 chunk = 1ull << 24;
  double *dl, *dc, *dn;
  cudaMalloc(&dl, 8 * chunk);
  cudaMalloc(&dc, 8 * chunk);
  cudaMalloc(&dn, 8 * chunk);
  std::vector<double> hl(chunk), hc(chunk), hn(chunk);
  u64 bad_log = 0, bad_cos = 0, bad_norm = 0, shown = 0;
  double max_ulp_norm = 0;
  for (u64 base = 0; base < n; base += chunk) {
    const u64 m = std::min(chunk, n - base);
    // positions 2 (base + i), 2 (base + i) + 1: the counter offset folded into the key
    k_draws<<<148 * 16, 256>>>(key + 2 * base * kGolden, m, dl, dc, dn);
    cudaMemcpy(hl.data(), dl, 8 * m, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc.data(), dc, 8 * m, cudaMemcpyDeviceToHost);
    cudaMemcpy(hn.data(), dn, 8 * m, cudaMemcpyDeviceToHost);
    for (u64 i = 0; i < m; ++i) {
      const u64 pos = 2 * (base + i);
      const double u1 = 1.0 - u01_at(key, pos);
      const double u2 = u01_at(key, pos + 1);
      const double l = std::log(u1), c = std::cos(2.0 * kPi * u2);
      const double v = std::sqrt(-2.0 * l) * c;
      const bool bl = bits(l) != bits(hl[i]), bc = bits(c) != bits(hc[i]), bn = bits(v) != bits(hn[i]);
      bad_log += bl;
      bad_cos += bc;
      bad_norm += bn;
      if (bn) {
        const double ulp = std::fabs(v - hn[i]) / std::fabs(std::nextafter(v, 2 * v) - v);
        if (ulp > max_ulp_norm) max_ulp_norm = ulp;
      }
      if ((bl || bc) && shown < 6) {
        ++shown;
        std::printf("draw %llu: u1=%.17g u2=%.17g  glibc log=%a cos=%a | device log=%a cos=%a\n",
                    (unsigned long long)(base + i), u1, u2, l, c, hl[i], hc[i]);
      }
    }
  }
  std::printf("draws %llu: log differs in %llu, cos differs in %llu, normal differs in %llu "
              "(max %.1f ulp)\n",
              (unsigned long long)n, (unsigned long long)bad_log, (unsigned long long)bad_cos,
              (unsigned long long)bad_norm, max_ulp_norm);
  return 0;
}
