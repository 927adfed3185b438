// Probe: CUDA graph conditional nodes (WHILE containing an upstream kernel and
// a SWITCH) built through stream capture, with PDL-attributed kernels inside
// the bodies.  Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_init(int* c, int M, cudaGraphConditionalHandle hw) {
  c[0] = 0;  // c0
  c[1] = M;
  c[2] = 0;  // iterations
  cudaGraphSetConditional(hw, M > 0 ? 1u : 0u);
}
__global__ void k_chunk(int* c, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs) {
  const int rem = c[1] - c[0];
  const int cs = rem > 32 ? 2 : (rem > 16 ? 1 : 0);  // chunk 64 / 32 / 16
  const int tc = 16 << cs;
  c[3] = c[0];
  c[0] += tc;
  c[2] += 1;
  cudaGraphSetConditional(hs, (unsigned)cs);
  cudaGraphSetConditional(hw, c[0] < c[1] ? 1u : 0u);
}
__global__ void k_work(int* c, int* acc, int tc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(acc, tc * 1000 + 1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static cudaError_t launch_pdl(void (*k)(int*, int*, int), cudaStream_t st, int* c, int* acc, int tc) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(32);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, c, acc, tc);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

int main() {
  int *c, *acc;
  CK(cudaMalloc(&c, 64));
  CK(cudaMalloc(&acc, 4));
  cudaStream_t st, st2;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  int Mh = 0;
  CK(cudaMemcpy(acc, &Mh, 4, cudaMemcpyHostToDevice));
  for (int M : {0, 10, 40, 100}) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    CK(launch_pdl(k_work, st, c, acc, 0));  // upstream PDL kernel
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps;
    size_t nd;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphConditionalHandle hw;
    CK(cudaGraphConditionalHandleCreate(&hw, cg, 0, 0));
    k_init<<<1, 1, 0, st>>>(c, M, hw);
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, cg, deps, nd, &wp));
    CK(cudaStreamUpdateCaptureDependencies(st, &wnode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    // body: k_chunk then SWITCH over 3 chunk sizes
    cudaGraphConditionalHandle hs;
    CK(cudaGraphConditionalHandleCreate(&hs, body, 0, 0));
    CK(cudaStreamBeginCaptureToGraph(st2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_chunk<<<1, 1, 0, st2>>>(c, hw, hs);
    CK(cudaStreamGetCaptureInfo(st2, &cs, nullptr, nullptr, &deps, &nd));
    cudaGraphNodeParams sp = {};
    sp.type = cudaGraphNodeTypeConditional;
    sp.conditional.handle = hs;
    sp.conditional.type = cudaGraphCondTypeSwitch;
    sp.conditional.size = 3;
    cudaGraphNode_t snode;
    CK(cudaGraphAddNode(&snode, body, deps, nd, &sp));
    CK(cudaStreamUpdateCaptureDependencies(st2, &snode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(st2, &tmp));
    for (int k = 0; k < 3; ++k) {
      CK(cudaStreamBeginCaptureToGraph(st2, sp.conditional.phGraph_out[k], nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      CK(launch_pdl(k_work, st2, c, acc, 16 << k));
      CK(launch_pdl(k_work, st2, c, acc, 16 << k));
      CK(cudaStreamEndCapture(st2, &tmp));
    }
    CK(launch_pdl(k_work, st, c, acc, 0));  // downstream
    CK(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, graph, 0));
    int z = 0;
    CK(cudaMemcpy(acc, &z, 4, cudaMemcpyHostToDevice));
    CK(cudaGraphLaunch(ex, st));
    CK(cudaGraphLaunch(ex, st));
    CK(cudaStreamSynchronize(st));
    int h[4], a;
    CK(cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&a, acc, 4, cudaMemcpyDeviceToHost));
    printf("M=%d iterations=%d acc=%d\n", M, h[2], a);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(graph);
  }
  printf("PROBE OK\n");
  return 0;
}
