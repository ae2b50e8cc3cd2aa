// tc_host.cu -- weight repacks into K-major bf16 layouts for TMA/UMMA, capability check,
// and the history projection driver of the bf16 path.
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "launch.h"
#include "tc.h"

namespace stca {

static __global__ void k_transpose_bf16(const bf16 *__restrict__ src, int64_t rows, int64_t cols,
                                        bf16 *__restrict__ dst) {
  __shared__ bf16 t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) t[i][threadIdx.x] = src[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;  // dst [cols x rows]
    if (r < rows && c < cols) dst[c * rows + r] = t[threadIdx.x][i];
  }
}

static void *transpose_dev(const void *src, int64_t rows, int64_t cols, const DevAlloc &alloc) {
  void *dst = alloc((size_t)rows * cols * 2);
  if (!dst) return nullptr;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  note_launch();
  k_transpose_bf16<<<grid, dim3(32, 8)>>>((const bf16 *)src, rows, cols, (bf16 *)dst);
  if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
  return dst;
}

static uint16_t to_bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

// ---- per-device caches (every entry keyed by the current device ordinal) ----
static std::mutex g_dev_mu;
static std::map<std::pair<const void *, int>, int> g_optin, g_occ;
static std::map<int, int> g_sms, g_tc_ok;

static int cur_dev() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}

cudaError_t smem_optin(const void *kernel, int bytes) {
  const int dev = cur_dev();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  int &done = g_optin[{kernel, dev}];
  if (done >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done = bytes;
  return e;
}

int sm_count() {
  const int dev = cur_dev();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  int &n = g_sms[dev];
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 1;
    }
  }
  return n;
}

int cluster_occupancy(const void *kernel, int threads, int smem, int cluster) {
  const int dev = cur_dev();
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_occ.find({kernel, dev});
    if (it != g_occ.end()) return it->second;
  }
  int mc = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cluster);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cudaLaunchAttribute ca[1];
  ca[0].id = cudaLaunchAttributeClusterDimension;
  ca[0].val.clusterDim.x = (unsigned)cluster;
  ca[0].val.clusterDim.y = 1;
  ca[0].val.clusterDim.z = 1;
  cfg.attrs = ca;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&mc, kernel, &cfg) != cudaSuccess || mc <= 0) {
    cudaGetLastError();
    mc = std::max(1, sm_count() / cluster);
  }
  std::lock_guard<std::mutex> lk(g_dev_mu);
  g_occ[{kernel, dev}] = mc;
  return mc;
}

bool tc_available() {
  const int dev = cur_dev();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_tc_ok.find(dev);
  if (it != g_tc_ok.end()) return it->second == 1;
  int major = 0, minor = 0;
  const bool ok = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess &&
                  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess &&
                  major == 10 && minor == 0;
  cudaGetLastError();
  g_tc_ok[dev] = ok ? 1 : 0;
  return ok;
}

bool tc_prepare_ffn(const float *Wu, const float *Wv, const float *Wo, int d, int rd, TcWeights *tc,
                    const DevAlloc &alloc) {
  // W1^T [2rd x d], 32-row chunks interleaved: rows 64c..64c+31 = Wu[:, 32c..]^T, +32.. = Wv[:, 32c..]^T
  std::vector<uint16_t> w1((size_t)2 * rd * d), wo((size_t)d * rd);
  for (int c = 0; c < rd / 32; ++c)
    for (int j = 0; j < 32; ++j)
      for (int e = 0; e < d; ++e) {
        w1[(size_t)(64 * c + j) * d + e] = to_bf16_bits(Wu[(size_t)e * rd + 32 * c + j]);
        w1[(size_t)(64 * c + 32 + j) * d + e] = to_bf16_bits(Wv[(size_t)e * rd + 32 * c + j]);
      }
  for (int k = 0; k < rd; ++k)
    for (int n = 0; n < d; ++n) wo[(size_t)n * rd + k] = to_bf16_bits(Wo[(size_t)k * d + n]);
  tc->W1h = alloc(w1.size() * 2);
  tc->Woh = alloc(wo.size() * 2);
  if (!tc->W1h || !tc->Woh) return false;
  return cudaMemcpy(tc->W1h, w1.data(), w1.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(tc->Woh, wo.data(), wo.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess;
}

bool tc_prepare_layer(const void *WQK, const void *WVO, const void *WC, int i, int d, int h, TcWeights *tc,
                      const DevAlloc &alloc) {
  if (WQK && !(tc->WQK = transpose_dev(WQK, d, (int64_t)h * d, alloc))) return false;
  if (WVO && !(tc->WVO = transpose_dev(WVO, (int64_t)h * d, d, alloc))) return false;
  if (WC && !(tc->WC = transpose_dev(WC, (int64_t)i * d, d, alloc))) return false;
  return true;
}

}  // namespace stca

namespace stca {

bool tc_prepare_proj(const float *const *Wu, const float *const *Wv, const float *const *Wo, const float *const *g,
                     const float *const *b, int M, int d, int rd, TcProjWeights *out, const DevAlloc &alloc) {
  std::vector<uint16_t> w1((size_t)M * 2 * rd * d), wo((size_t)M * rd * d);
  std::vector<float> gg((size_t)M * d), bb((size_t)M * d);
  for (int i = 0; i < M; ++i) {
    uint16_t *W1 = w1.data() + (size_t)i * 2 * rd * d, *WO = wo.data() + (size_t)i * rd * d;
    // fused projection: 64-column chunks, rows 128c..128c+63 = Wu[:, 64c..]^T, +64.. = Wv[:, 64c..]^T
    for (int c = 0; c < rd / 64; ++c)
      for (int j = 0; j < 64; ++j)
        for (int e = 0; e < d; ++e) {
          W1[(size_t)(128 * c + j) * d + e] = to_bf16_bits(Wu[i][(size_t)e * rd + 64 * c + j]);
          W1[(size_t)(128 * c + 64 + j) * d + e] = to_bf16_bits(Wv[i][(size_t)e * rd + 64 * c + j]);
        }
    for (size_t k = 0; k < (size_t)rd * d; ++k) WO[k] = to_bf16_bits(Wo[i][k]);
    memcpy(gg.data() + (size_t)i * d, g[i], sizeof(float) * d);
    memcpy(bb.data() + (size_t)i * d, b[i], sizeof(float) * d);
  }
  out->W1cat = alloc(w1.size() * 2);
  out->Wocat = alloc(wo.size() * 2);
  out->gcat = (float *)alloc(gg.size() * 4);
  out->bcat = (float *)alloc(bb.size() * 4);
  if (!out->W1cat || !out->Wocat || !out->gcat || !out->bcat) return false;
  return cudaMemcpy(out->W1cat, w1.data(), w1.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(out->Wocat, wo.data(), wo.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(out->gcat, gg.data(), gg.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(out->bcat, bb.data(), bb.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
}

}  // namespace stca
