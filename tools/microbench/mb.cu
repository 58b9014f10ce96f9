// Microbenchmarks for the B200 design decisions of the Log-Fourier SP decoder
// (FP32 FFMA vs FFMA2 issue rate, MUFU ex2/lg2 rate, LDS.128 rate, HBM and L2
// read bandwidth, launch gaps, CUDA-graph WHILE conditional nodes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo mb.cu -o mb
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void ffma_tp(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float y0 = a + threadIdx.x, y1 = b - threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fmaf(x0, y0, y1); x1 = fmaf(x1, y1, y0); x2 = fmaf(x2, y0, y1); x3 = fmaf(x3, y1, y0);
      x4 = fmaf(x4, y0, y1); x5 = fmaf(x5, y1, y0); x6 = fmaf(x6, y0, y1); x7 = fmaf(x7, y1, y0);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ffma2_tp(float* out, int iters, float a, float b) {
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, threadIdx.x), x2 = make_float2(3, 4), x3 = make_float2(5, 6);
  float2 x4 = make_float2(7, 8), x5 = make_float2(9, 10), x6 = make_float2(11, 12), x7 = make_float2(13, 14);
  float s0 = a + threadIdx.x, s1 = b - threadIdx.x;
  float2 c = make_float2(a, b);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = __ffma2_rn(make_float2(s0, s0), x0, c); x1 = __ffma2_rn(make_float2(s1, s1), x1, c);
      x2 = __ffma2_rn(make_float2(s0, s0), x2, c); x3 = __ffma2_rn(make_float2(s1, s1), x3, c);
      x4 = __ffma2_rn(make_float2(s0, s0), x4, c); x5 = __ffma2_rn(make_float2(s1, s1), x5, c);
      x6 = __ffma2_rn(make_float2(s0, s0), x6, c); x7 = __ffma2_rn(make_float2(s1, s1), x7, c);
    }
  }
  float2 r = make_float2(x0.x + x1.x + x2.x + x3.x + x4.x + x5.x + x6.x + x7.x, x0.y + x1.y + x2.y + x3.y + x4.y + x5.y + x6.y + x7.y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r.x + r.y;
}

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2a(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void ex2_tp(float* out, int iters) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = -0.001f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ex2a(x[j]) - 1.0f;
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lg2_tp(float* out, int iters) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = 1.5f + 0.001f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = lg2a(x[j]) + 2.0f;
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void lds128_tp(float* out, int iters) {
  __shared__ float4 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x & 31;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 v = sm[(idx + j * 32 + i) & 1023];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void read_bw(const float4* __restrict__ in, size_t n, int reps, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      float4 v = in[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = 1;
}
__global__ void write_bw(float4* out, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) out[i] = make_float4(1, 2, 3, 4);
}

__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 12345) p[0] = 1; }

__global__ void while_body(int* counter, int limit, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int c = ++counter[0];
    if (c >= limit) cudaGraphSetConditional(h, 0);
  }
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"smem_optin\": %zu}\n", prop.name, prop.multiProcessorCount, clk, prop.l2CacheSize, prop.sharedMemPerMultiprocessor, prop.sharedMemPerBlockOptin);
  int sms = prop.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, 64 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // FFMA
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4096; int blocks = sms * 8, threads = 256;
    ffma_tp<<<blocks, threads>>>(out, 16, 1.0001f, 0.5f);
    cudaEventRecord(e0); ffma_tp<<<blocks, threads>>>(out, iters, 1.0001f, 0.5f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * threads * iters * 64;
    printf("{\"test\": \"ffma\", \"fma_per_s\": %.4e, \"per_sm_per_clk_at_max\": %.2f, \"ms\": %.3f}\n", fma / (ms * 1e-3), fma / (ms * 1e-3) / sms / (clk * 1e3), ms);
    ffma2_tp<<<blocks, threads>>>(out, 16, 1.0001f, 0.5f);
    cudaEventRecord(e0); ffma2_tp<<<blocks, threads>>>(out, iters, 1.0001f, 0.5f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fma = (double)blocks * threads * iters * 64 * 2;
    printf("{\"test\": \"ffma2\", \"fma_per_s\": %.4e, \"per_sm_per_clk_at_max\": %.2f, \"ms\": %.3f}\n", fma / (ms * 1e-3), fma / (ms * 1e-3) / sms / (clk * 1e3), ms);
  }
  {
    int iters = 2048; int blocks = sms * 8, threads = 256;
    ex2_tp<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); ex2_tp<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 8;
    printf("{\"test\": \"ex2\", \"ops_per_s\": %.4e, \"per_sm_per_clk_at_max\": %.2f}\n", ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3));
    lg2_tp<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); lg2_tp<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"lg2\", \"ops_per_s\": %.4e, \"per_sm_per_clk_at_max\": %.2f}\n", ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    int iters = 2048; int blocks = sms * 8, threads = 256;
    lds128_tp<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); lds128_tp<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)blocks * threads * iters * 8 * 16;
    printf("{\"test\": \"lds128\", \"bytes_per_sm_per_clk_at_max\": %.2f}\n", bytes / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    size_t big = (size_t)4 << 30; float4* buf; CK(cudaMalloc(&buf, big));
    write_bw<<<sms * 8, 512>>>(buf, big / 16);
    cudaEventRecord(e0); write_bw<<<sms * 8, 512>>>(buf, big / 16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"hbm_write\", \"GBps\": %.1f}\n", big / (ms * 1e-3) / 1e9);
    read_bw<<<sms * 8, 512>>>(buf, big / 16, 1, out);
    cudaEventRecord(e0); read_bw<<<sms * 8, 512>>>(buf, big / 16, 1, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"hbm_read\", \"GBps\": %.1f}\n", big / (ms * 1e-3) / 1e9);
    for (size_t l2b : {(size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20}) {
      int reps = (int)(((size_t)8 << 30) / l2b);
      read_bw<<<sms * 8, 512>>>(buf, l2b / 16, 2, out);
      cudaEventRecord(e0); read_bw<<<sms * 8, 512>>>(buf, l2b / 16, reps, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"test\": \"l2_read\", \"MB\": %zu, \"GBps\": %.1f}\n", l2b >> 20, (double)l2b * reps / (ms * 1e-3) / 1e9);
    }
    cudaFree(buf);
  }
  {
    int n = 2000;
    for (int i = 0; i < 10; ++i) empty_kernel<<<sms, 128>>>(nullptr);
    cudaEventRecord(e0); for (int i = 0; i < n; ++i) empty_kernel<<<sms, 128>>>(nullptr); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"launch_stream\", \"us_per_kernel\": %.3f}\n", ms * 1e3 / n);
    // big grid of empty CTAs
    cudaEventRecord(e0); for (int i = 0; i < 100; ++i) empty_kernel<<<65536, 256>>>(nullptr); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"empty_grid_65536x256\", \"us_per_kernel\": %.3f}\n", ms * 1e3 / 100);
    // captured graph of n kernels
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 200; ++i) empty_kernel<<<sms, 128, 0, s>>>(nullptr);
    CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s); for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"launch_graph\", \"us_per_kernel\": %.3f}\n", ms * 1e3 / 2000);
    // WHILE conditional
    int* counter; CK(cudaMalloc(&counter, 4));
    cudaGraph_t wg; CK(cudaGraphCreate(&wg, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, wg, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t cn; CK(cudaGraphAddNode(&cn, wg, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    int limit = 1000;
    void* args[] = {&counter, &limit, &h};
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    kp.kernel.func = (void*)while_body; kp.kernel.gridDim = dim3(sms); kp.kernel.blockDim = dim3(128); kp.kernel.kernelParams = args;
    cudaGraphNode_t kn; CK(cudaGraphAddNode(&kn, body, nullptr, 0, &kp));
    cudaGraphExec_t wge; CK(cudaGraphInstantiate(&wge, wg, 0));
    CK(cudaMemsetAsync(counter, 0, 4, s)); CK(cudaGraphLaunch(wge, s)); CK(cudaStreamSynchronize(s));
    CK(cudaMemsetAsync(counter, 0, 4, s));
    cudaEventRecord(e0, s); CK(cudaGraphLaunch(wge, s)); cudaEventRecord(e1, s); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    int hc; cudaMemcpy(&hc, counter, 4, cudaMemcpyDeviceToHost);
    printf("{\"test\": \"graph_while\", \"iters\": %d, \"us_per_iter\": %.3f}\n", hc, ms * 1e3 / hc);
  }
  return 0;
}
