// launch.h -- host helper: every decode-step kernel is launched through
// cudaLaunchKernelEx so that a launch can carry a scheduling priority (the
// sub-batch pipeline of api.cu gives the HBM-streaming block-score kernel the
// lowest priority and the latency-bound selection / attention kernels the
// highest, so that their CTAs are placed first whenever an SM frees up) and a
// thread-block cluster shape, and the token / attention kernels are launched
// with programmatic stream serialization (PDL) so that their CTAs start while
// the previous kernel drains; their data dependences are per-pair ready flags
// (common.cuh wait_ready).
#pragma once

#include <cuda_runtime.h>

#include <mutex>

namespace tls {

// cudaFuncSetAttribute is a host round trip; the decode step launches four
// kernels per call, so the attributes are set once per (kernel, device) and
// again only when a larger dynamic shared-memory size is needed.
static inline cudaError_t prepare_kernel(const void* kern, size_t smem, bool nonportable_cluster) {
  struct Entry {
    const void* k;
    int dev;
    size_t smem;
    bool np;
  };
  static Entry cache[256];
  static int n = 0;
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  int i = 0;
  for (; i < n; ++i)
    if (cache[i].k == kern && cache[i].dev == dev) break;
  if (i < n && cache[i].smem >= smem && (cache[i].np || !nonportable_cluster)) return cudaSuccess;
  const size_t want = (i < n && cache[i].smem > smem) ? cache[i].smem : smem;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  if (nonportable_cluster) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (i == n && n < 256) {
    cache[n++] = Entry{kern, dev, smem, nonportable_cluster};
  } else if (i < n) {
    cache[i].smem = smem > cache[i].smem ? smem : cache[i].smem;
    cache[i].np = cache[i].np || nonportable_cluster;
  }
  return cudaSuccess;
}

struct LaunchOpts {
  int prio = 0;     // cudaLaunchAttributePriority value (0 = default / lowest; more negative = higher)
  int use_prio = 0; // attach the priority attribute
  int pdl = 0;      // programmatic stream serialization: may start before the previous kernel finishes
};

template <typename P>
static inline cudaError_t launch_ex(void (*kern)(const P), dim3 grid, int threads, size_t smem, cudaStream_t st,
                                    const LaunchOpts& o, unsigned cluster_x, const P& p) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = dim3((unsigned)threads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (cluster_x > 0) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster_x;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (o.use_prio) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = o.prio;
    ++na;
  }
  if (o.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  lc.attrs = attr;
  lc.numAttrs = (unsigned)na;
  return cudaLaunchKernelEx(&lc, kern, p);
}

}  // namespace tls
