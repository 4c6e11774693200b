// Host-side copy probe (design aid): cost of pinning, pageable vs pinned D2H,
// and huge-page first touch for a solution-key sized transfer.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); }
int main() {
  const size_t n = 400ull << 20;
  void* d;
  cudaMalloc(&d, n);
  cudaMemset(d, 1, n);
  cudaDeviceSynchronize();
  auto t = clk::now();
  void* h;
  cudaHostAlloc(&h, n, cudaHostAllocDefault);
  printf("cudaHostAlloc 400MB: %.1f ms\n", ms(t));
  t = clk::now();
  cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost);
  printf("D2H pinned: %.1f ms\n", ms(t));
  t = clk::now();
  cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost);
  printf("D2H pinned again: %.1f ms\n", ms(t));
  for (int huge = 0; huge < 2; ++huge) {
    char* p = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
    if (huge) madvise(p, n, MADV_HUGEPAGE);
    t = clk::now();
    cudaMemcpy(p, d, n, cudaMemcpyDeviceToHost);
    printf("D2H pageable fresh (madv_huge=%d): %.1f ms\n", huge, ms(t));
    t = clk::now();
    cudaMemcpy(p, d, n, cudaMemcpyDeviceToHost);
    printf("D2H pageable touched (madv_huge=%d): %.1f ms\n", huge, ms(t));
    char* q = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
    if (huge) madvise(q, n, MADV_HUGEPAGE);
    t = clk::now();
    memcpy(q, h, n);
    printf("memcpy pinned->fresh (huge=%d): %.1f ms\n", huge, ms(t));
    char* r = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
    if (huge) madvise(r, n, MADV_HUGEPAGE);
    t = clk::now();
    std::vector<std::thread> th;
    const int T = 8;
    for (int i = 0; i < T; ++i) th.emplace_back([&, i] { memcpy(r + n / T * i, static_cast<char*>(h) + n / T * i, n / T); });
    for (auto& x : th) x.join();
    printf("memcpy x8 threads pinned->fresh (huge=%d): %.1f ms\n", huge, ms(t));
    t = clk::now();
    cudaHostRegister(r, n, cudaHostRegisterDefault);
    printf("cudaHostRegister touched (huge=%d): %.1f ms\n", huge, ms(t));
    t = clk::now();
    cudaMemcpy(r, d, n, cudaMemcpyDeviceToHost);
    printf("D2H registered: %.1f ms\n", ms(t));
    cudaHostUnregister(r);
  }
  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  char buf[256] = {0};
  if (f && fgets(buf, sizeof buf, f)) printf("THP: %s", buf);
  printf("cores: %u\n", std::thread::hardware_concurrency());
  return 0;
}
