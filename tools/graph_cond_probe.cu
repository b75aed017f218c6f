// graph_cond_probe.cu — does this driver/runtime run a WHILE conditional node whose body holds an
// IF conditional node, with both handles (and a third, the body's) set from kernels nested inside
// the IF body?  (The device-resident eigensolver loop of k_eig.cu relies on it.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/gcp tools/graph_cond_probe.cu && /tmp/gcp
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// top of the body: iteration counter; sets the body's IF handles from device state (so their
// values never depend on when a body-owned handle's default would be applied)
__global__ void k_inc(int* st, cudaGraphConditionalHandle hif, cudaGraphConditionalHandle hpow) {
  if (threadIdx.x == 0) {
    st[0] += 1;
    cudaGraphSetConditional(hif, st[3] ? 1u : 0u);
    cudaGraphSetConditional(hpow, 1u);
  }
}
__global__ void k_ctl_if(int* st, cudaGraphConditionalHandle hloop, cudaGraphConditionalHandle hpow) {
  // runs inside the IF body: every 3rd iteration; stops the loop at iteration >= 10
  if (threadIdx.x == 0) {
    st[1] += 1;
    if (st[0] >= 10) { cudaGraphSetConditional(hloop, 0); cudaGraphSetConditional(hpow, 0); }
    else cudaGraphSetConditional(hpow, 1);
  }
}
__global__ void k_pow(int* st) { if (threadIdx.x == 0) st[2] += 1; }
__global__ void k_step(int* st) {
  if (threadIdx.x == 0) st[3] = ((st[0] + 1) % 3 == 0) ? 1 : 0;  // IF fires in iterations 3, 6, 9, 12
}

__global__ void k_count(int* st, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0 && ++st[0] >= 100) cudaGraphSetConditional(h, 0);
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  int* st;
  CK(cudaMalloc(&st, 16));
  CK(cudaMemset(st, 0, 16));
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hloop;
  CK(cudaGraphConditionalHandleCreate(&hloop, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hloop;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hif, hpow;
  CK(cudaGraphConditionalHandleCreate(&hif, body, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hpow, body, 0, 0));
  // body: inc -> IF(hif){ctl_if} -> IF(hpow){pow -> step}
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_inc<<<1, 32, 0, s>>>(st, hif, hpow);
  CK(cudaStreamEndCapture(s, &body));
  cudaGraphNode_t inc_node;
  size_t n = 1;
  CK(cudaGraphGetNodes(body, &inc_node, &n));
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hif;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 1;
  cudaGraphNode_t ifnode;
  CK(cudaGraphAddNode(&ifnode, body, &inc_node, 1, &ip));
  cudaGraph_t ifbody = ip.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, ifbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_ctl_if<<<1, 32, 0, s>>>(st, hloop, hpow);
  CK(cudaStreamEndCapture(s, &ifbody));
  cudaGraphNodeParams pp = {};
  pp.type = cudaGraphNodeTypeConditional;
  pp.conditional.handle = hpow;
  pp.conditional.type = cudaGraphCondTypeIf;
  pp.conditional.size = 1;
  cudaGraphNode_t pnode;
  CK(cudaGraphAddNode(&pnode, body, &ifnode, 1, &pp));
  cudaGraph_t pbody = pp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, pbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_pow<<<1, 32, 0, s>>>(st);
  k_step<<<1, 32, 0, s>>>(st);
  CK(cudaStreamEndCapture(s, &pbody));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemsetAsync(st, 0, 16, s));  // st[3] = 0: no IF in iteration 1
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    int h[4];
    CK(cudaMemcpy(h, st, 16, cudaMemcpyDeviceToHost));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // expected: IF (ctl) in iterations 3, 6, 9, 12; the one at 12 (>= 10) stops the loop before
    // pow: iters=12 ctl=4 pow=11
    printf("rep %d: iters=%d ctl=%d pow=%d  (%.1f us total, %.2f us/iter)\n", rep, h[0], h[1], h[2], ms * 1e3,
           ms * 1e3 / (h[0] > 0 ? h[0] : 1));
  }
  // node overhead: WHILE body of 10 dependent empty kernels (the last counts down), 100 iterations
  {
    cudaGraph_t g2;
    CK(cudaGraphCreate(&g2, 0));
    cudaGraphConditionalHandle h2;
    CK(cudaGraphConditionalHandleCreate(&h2, g2, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams w2 = {};
    w2.type = cudaGraphNodeTypeConditional;
    w2.conditional.handle = h2;
    w2.conditional.type = cudaGraphCondTypeWhile;
    w2.conditional.size = 1;
    cudaGraphNode_t n2;
    CK(cudaGraphAddNode(&n2, g2, nullptr, 0, &w2));
    cudaGraph_t b2 = w2.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, b2, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < 9; ++i) k_pow<<<148, 128, 0, s>>>(st + 3);
    k_count<<<1, 32, 0, s>>>(st, h2);
    CK(cudaStreamEndCapture(s, &b2));
    cudaGraphExec_t ge2;
    CK(cudaGraphInstantiate(&ge2, g2, 0));
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemsetAsync(st, 0, 16, s));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      CK(cudaGraphLaunch(ge2, s));
      cudaEventRecord(e1, s);
      CK(cudaStreamSynchronize(s));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("while x100 of 10 kernel nodes: %.1f us -> %.2f us per node\n", ms * 1e3, ms * 1e3 / 1000);
    }
    // same 1000 launches from the host, stream-ordered
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 1000; ++i) k_pow<<<148, 128, 0, s>>>(st + 3);
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("1000 host launches: %.1f us -> %.2f us per launch\n", ms * 1e3, ms * 1e3 / 1000);
  }
  printf("OK\n");
  return 0;
}
