// L2 warm-up probe: does a region pulled into L2 ahead of time (bulk prefetch,
// or plain loads with an evict_last policy) make a later streaming read of the
// same bytes faster?  Region = `rows` rows of `row_bytes` from a larger buffer
// (stride `stride` bytes), like the first k-blocks of an expert's weight tiles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_warm l2_warm.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void warm_bulk(const char* base, long long stride, int rows, int row_bytes) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + (long long)i * stride), "r"(row_bytes)
                 : "memory");
}

__global__ void warm_ld(const char* base, long long stride, int rows, int row_bytes, int* sink) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const int v_per_row = row_bytes / 16;
  const long long n = (long long)rows * v_per_row;
  int acc = 0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long r = j / v_per_row, c = j % v_per_row;
    const char* p = base + r * stride + c * 16;
    int4 v;
    asm volatile("ld.global.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    acc ^= v.x;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

__global__ void warm_prefetch_ld(const char* base, long long stride, int rows, int row_bytes) {
  const int lines = row_bytes / 128;
  const long long n = (long long)rows * lines;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long r = j / lines, c = j % lines;
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(base + r * stride + c * 128));
  }
}

__global__ void stream_read(const char* base, long long stride, int rows, int row_bytes, int* sink, int evict_first) {
  uint64_t pol;
  if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  const int v_per_row = row_bytes / 16;
  const long long n = (long long)rows * v_per_row;
  int acc = 0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long r = j / v_per_row, c = j % v_per_row;
    int4 v;
    asm volatile("ld.global.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(base + r * stride + c * 16), "l"(pol));
    acc ^= v.x;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

__global__ void flush(char* buf, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n / 16; i += (long long)gridDim.x * blockDim.x)
    reinterpret_cast<int4*>(buf)[i] = make_int4(i, 0, 0, 0);
}

int main() {
  const long long stride = 28672;  // Mixtral gate row (f = 14336 bf16)
  const int row_bytes = 28672;
  const long long total = 512LL << 20;
  char *buf, *fl;
  int* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&fl, 512LL << 20);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"none", "bulk", "ld_evict_last", "prefetch_evict_last"};
  for (int mb : {32, 64, 96}) {
    const int rows = (int)(((long long)mb << 20) / row_bytes);
    for (int ef = 0; ef < 2; ++ef) {
      for (int mode = 0; mode < 4; ++mode) {
        float best = 1e9, wtime = 0;
        for (int rep = 0; rep < 5; ++rep) {
          flush<<<1184, 256>>>(fl, 512LL << 20);
          cudaEventRecord(a);
          if (mode == 1) warm_bulk<<<(rows + 63) / 64, 64>>>(buf, stride, rows, row_bytes);
          if (mode == 2) warm_ld<<<1184, 256>>>(buf, stride, rows, row_bytes, sink);
          if (mode == 3) warm_prefetch_ld<<<1184, 256>>>(buf, stride, rows, row_bytes);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float w;
          cudaEventElapsedTime(&w, a, b);
          cudaEventRecord(a);
          stream_read<<<148 * 4, 256>>>(buf, stride, rows, row_bytes, sink, ef);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) { best = ms; wtime = w; }
        }
        printf("%3d MB read(evict_first=%d) after %-20s: %7.1f us  (%6.0f GB/s)  warm kernel %7.1f us\n", mb, ef,
               names[mode], best * 1e3, (double)rows * row_bytes / (best * 1e-3) / 1e9, wtime * 1e3);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
