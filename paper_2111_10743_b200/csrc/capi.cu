// C-ABI bookkeeping: last-error string, version, device query.
#include <cstring>
#include <string>
#include <vector>

#include "lb_common.cuh"

namespace lb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int sm_count() {
  static int cached = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cached < 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached = n;
  }
  return cached;
}

}  // namespace lb

extern "C" {

int lb_abi_version(void) { return LB_ABI_VERSION; }

const char* lb_last_error_string(void) { return lb::g_last_error.c_str(); }

/* Kernel nodes of a captured CUDA graph (cudaGraph_t passed as void*): the
 * bench's count of the library's launches inside one replayed step. */
int lb_graph_kernel_nodes(void* graph, int64_t* nkernels, int64_t* nnodes) {
  if (!graph || !nkernels) return lb::fail(LB_ERR_ARG, "lb_graph_kernel_nodes: null argument");
  cudaGraph_t g = (cudaGraph_t)graph;
  size_t n = 0;
  LB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) LB_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
  int64_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    LB_CUDA(cudaGraphNodeGetType(nodes[i], &t));
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  *nkernels = k;
  if (nnodes) *nnodes = (int64_t)n;
  return LB_OK;
}

int lb_device_info(int* sms, int* major, int* minor) {
  int dev = 0;
  LB_CUDA(cudaGetDevice(&dev));
  if (sms) LB_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  if (major) LB_CUDA(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev));
  if (minor) LB_CUDA(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev));
  return LB_OK;
}

}  // extern "C"
