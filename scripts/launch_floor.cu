// launch_floor.cu -- the floor of an event-bracketed kernel launch on B200
// (diagnostic only): an empty kernel with the GEMM's launch shape (148 CTAs x
// 192 threads, 193 KB dynamic shared memory), the same without shared memory,
// and a 1-CTA kernel; each timed (a) bracketed alone by two CUDA events, as
// bench.py's per-launch roofline pass does, (b) 100 back to back, (c) 100
// back to back with programmatic dependent launch (the kernel triggers its
// dependents first, then waits), (d) the PDL chain of (c) as one CUDA graph;
// and a graph chain of kernels that each spin 5 us with the dependent launch
// triggered at the start vs at the end (what an early trigger buys).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/launch_floor scripts/launch_floor.cu
#include <cstdio>

#include <cuda_runtime.h>

__global__ void k_empty() {
  extern __shared__ unsigned char s[];
  if (threadIdx.x == 1023) s[0] = 0;  // never true: keeps the shared-memory reservation
}

__global__ void k_empty_pdl() {
  extern __shared__ unsigned char s[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 1023) s[0] = 0;
}

static void launch_pdl(int grid, int block, int smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_empty_pdl);
}

static void run(const char* name, int grid, int block, int smem) {
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 10; ++i) k_empty<<<grid, block, smem>>>();
  cudaDeviceSynchronize();
  float iso = 0.f;
  for (int i = 0; i < 100; ++i) {
    cudaEventRecord(a);
    k_empty<<<grid, block, smem>>>();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    iso += ms;
  }
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) k_empty<<<grid, block, smem>>>();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float btb;
  cudaEventElapsedTime(&btb, a, b);
  cudaFuncSetAttribute(k_empty_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int i = 0; i < 10; ++i) launch_pdl(grid, block, smem, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(a, st);
  for (int i = 0; i < 100; ++i) launch_pdl(grid, block, smem, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float pdl;
  cudaEventElapsedTime(&pdl, a, b);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 100; ++i) launch_pdl(grid, block, smem, st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float gr;
  cudaEventElapsedTime(&gr, a, b);
  printf("%-40s isolated %6.2f us   back-to-back %6.2f us   PDL %6.2f us   PDL graph %6.2f us  (%s)\n", name,
         iso * 10.f, btb * 10.f, pdl * 10.f, gr * 10.f, cudaGetErrorString(cudaGetLastError()));
}

__global__ void k_spin(long long ns, int trig_first) {
  extern __shared__ unsigned char s[];
  if (trig_first) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (!trig_first) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 1023) s[0] = 0;
}

static void spin_chain(int smem, int trig_first) {
  cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 100; ++i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = 148;
    cfg.blockDim = 192;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_spin, 5000LL, trig_first);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("graph chain of 5 us spins, 148 x 192, %3d KB smem, trigger at %s: %6.2f us per kernel (%s)\n", smem / 1024,
         trig_first ? "start" : "end  ", ms * 10.f, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  spin_chain(193 * 1024, 1);
  spin_chain(193 * 1024, 0);
  spin_chain(0, 1);
  spin_chain(0, 0);
  run("148 x 192, 193 KB smem (GEMM shape)", 148, 192, 193 * 1024);
  run("148 x 192, no smem", 148, 192, 0);
  run("512 x 128, 38 KB smem (attention shape)", 512, 128, 38 * 1024);
  run("1 x 32", 1, 32, 0);
  return 0;
}
