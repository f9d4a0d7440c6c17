// Host cost of a kernel launch vs the size of its parameter block (diagnostics
// for the scheduler round's launch): cudaLaunchKernel wall time per call and
// launch-to-completion latency, for 64 B .. 4 KB of parameters.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

template <int BYTES>
struct P { unsigned char b[BYTES]; };

template <int BYTES>
__global__ void k(P<BYTES> p, int* out) {
  if (threadIdx.x == 0) *out = p.b[BYTES - 1];
}

template <int BYTES>
void run(int* d) {
  P<BYTES> p{};
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 200; ++i) k<BYTES><<<1, 512, 0, s>>>(p, d);
  cudaStreamSynchronize(s);
  double launch = 0, total = 0;
  const int n = 2000;
  for (int i = 0; i < n; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    k<BYTES><<<1, 512, 0, s>>>(p, d);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    launch += std::chrono::duration<double, std::micro>(t1 - t0).count();
    total += std::chrono::duration<double, std::micro>(t2 - t0).count();
  }
  std::printf("{\"param_bytes\": %d, \"launch_call_us\": %.2f, \"launch_to_sync_us\": %.2f}\n", BYTES, launch / n,
              total / n);
  cudaStreamDestroy(s);
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  run<64>(d);
  run<512>(d);
  run<1024>(d);
  run<1536>(d);
  run<2048>(d);
  run<4000>(d);
  return 0;
}
