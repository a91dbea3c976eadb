// Latency micro-benchmarks that size the cycle's launch structure on B200:
//  (1) back-to-back empty kernels captured in a CUDA graph,
//  (2) one cluster kernel doing K cluster barriers,
//  (3) one cluster kernel doing K phases of dependent L2 round trips.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 1000000) *p = 1;
}

__global__ void __launch_bounds__(256) k_bar(int k) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < k; ++i) cl.sync();
}

__global__ void __launch_bounds__(256) k_bar_relaxed(int k) {
  for (int i = 0; i < k; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
}

// each phase: every thread reads 8 values written by other CTAs in the previous phase
__global__ void __launch_bounds__(256) k_phases(double* buf, int n, int k) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = cl.block_rank() * blockDim.x + threadIdx.x, nthr = cl.num_blocks() * blockDim.x;
  for (int ph = 0; ph < k; ++ph) {
    double* src = buf + (size_t)(ph & 1) * n;
    double* dst = buf + (size_t)((ph + 1) & 1) * n;
    for (int v = tid; v < n; v += nthr) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += __ldcg(src + (v * 7 + q * 131) % n);
      dst[v] = s * 0.125;
    }
    cl.sync();
  }
}

float time_graph(cudaStream_t s, cudaGraphExec_t ge, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;  // us per graph
}

template <class F>
float time_capture(cudaStream_t s, F body, int reps = 200) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  body();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  float us = time_graph(s, ge, reps);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return us;
}

void launch_cluster(cudaStream_t s, void (*kern)(int), int cs, int k) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cs);
  lc.blockDim = dim3(256);
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaLaunchKernelEx(&lc, kern, k);
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaFuncSetAttribute(k_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_bar_relaxed, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_phases, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int nk : {1, 10}) {
    float us = time_capture(s, [&] { for (int i = 0; i < nk; ++i) k_empty<<<1, 32, 0, s>>>(nullptr); });
    printf("graph of %2d empty 1-block kernels: %.2f us/graph (%.2f us/kernel)\n", nk, us, us / nk);
    us = time_capture(s, [&] { for (int i = 0; i < nk; ++i) k_empty<<<2048, 256, 0, s>>>(nullptr); });
    printf("graph of %2d empty 2048-block kernels: %.2f us/graph (%.2f us/kernel)\n", nk, us, us / nk);
  }
  for (int cs : {8, 16}) {
    for (int k : {0, 8, 64}) {
      float us = time_capture(s, [&] { launch_cluster(s, k_bar, cs, k); });
      float ur = time_capture(s, [&] { launch_cluster(s, k_bar_relaxed, cs, k); });
      printf("cluster %2d, %2d cluster.sync: %.2f us (relaxed barrier %.2f us)\n", cs, k, us, ur);
    }
  }
  double* buf;
  cudaMalloc(&buf, 2 * 65536 * sizeof(double));
  cudaMemset(buf, 0, 2 * 65536 * sizeof(double));
  for (int n : {16, 784, 6724, 59536}) {
    for (int k : {1, 8}) {
      float us = time_capture(s, [&] {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(16);
        lc.blockDim = dim3(256);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, k_phases, buf, n, k);
      });
      printf("cluster 16 phases: n=%6d k=%d  %.2f us (%.2f us/phase)\n", n, k, us, us / k);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
