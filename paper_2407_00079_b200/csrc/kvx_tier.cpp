// kvx_tier.cpp -- the CPU-DRAM KVCache tier: layer-wise load (DRAM -> HBM) of
// a matched prefix and layer-wise store (HBM -> DRAM) of freshly computed KV,
// with Mooncake's launch / wait per layer: before a layer's
// attention the prefill waits for that layer's load; after it, the layer's
// store is launched; at the end all stores are waited for.  The reference
// models the effect as max(compute, cache load) (layerwise_effective_prefill,
// proj/src/perf_model.cpp:73-78) with load time = cached tokens x
// kv_bytes_per_token / load_bandwidth (cache_load_time, perf_model.cpp:80-85;
// load_bandwidth preset 30 GB/s, proj/src/config.cpp:218).  Here the bytes
// really move: the DRAM pool is pinned, device-mapped host memory in the same
// paged layout as HBM.  Scattered blocks: each layer is ONE copy kernel with a
// small grid (host_copy_ctas) that reads / writes it over PCIe, no staging.
// Contiguous block runs (kvx_layer_*_range): two copy-engine copies per
// layer and no kernel, so the SMs stay entirely with the prefill (a
// register-heavy GEMM leaves no room for a copy kernel beside it: bench.py's
// host_tier object measures both).  Loads and stores each have their own
// in-order queue, so a layer's load overlaps the previous layer's attention
// and its store overlaps the next layer's.
#include <cuda_runtime.h>

#include <vector>

#include "kvx.h"
#include "kvx_common.cuh"

using kvx::as_stream;

struct kvx_layer_io {
  int device = 0;
  int32_t max_layers = 0;
  cudaStream_t load_q = nullptr, store_q = nullptr;
  std::vector<cudaEvent_t> loaded;  // per layer: after that layer's last load
  cudaEvent_t dep = nullptr, stored = nullptr;
};

namespace {
int order_after(kvx_layer_io* io, cudaStream_t q, void* after) {
  if (!after) return KVX_OK;
  KVX_CUDA(cudaEventRecord(io->dep, as_stream(after)));
  KVX_CUDA(cudaStreamWaitEvent(q, io->dep, 0));
  return KVX_OK;
}
}  // namespace

extern "C" {

int kvx_layer_io_create(int device, int32_t max_layers, kvx_layer_io** out) {
  KVX_REQUIRE(out && max_layers >= 1, "kvx_layer_io_create: bad arguments");
  kvx::DeviceGuard g(device);
  auto* io = new kvx_layer_io();
  io->device = device;
  io->max_layers = max_layers;
  auto fail = [&](cudaError_t e) {
    kvx_layer_io_destroy(io);
    return kvx::cuda_error(e, "kvx_layer_io_create");
  };
  cudaError_t e = cudaStreamCreateWithFlags(&io->load_q, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&io->store_q, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&io->dep, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&io->stored, cudaEventDisableTiming);
  io->loaded.assign(max_layers, nullptr);
  for (int32_t l = 0; l < max_layers && e == cudaSuccess; ++l)
    e = cudaEventCreateWithFlags(&io->loaded[l], cudaEventDisableTiming);
  if (e != cudaSuccess) return fail(e);
  *out = io;
  return KVX_OK;
}

int kvx_layer_io_destroy(kvx_layer_io* io) {
  if (!io) return KVX_OK;
  kvx::DeviceGuard g(io->device);
  if (io->load_q) cudaStreamSynchronize(io->load_q);
  if (io->store_q) cudaStreamSynchronize(io->store_q);
  for (auto ev : io->loaded)
    if (ev) cudaEventDestroy(ev);
  if (io->dep) cudaEventDestroy(io->dep);
  if (io->stored) cudaEventDestroy(io->stored);
  if (io->load_q) cudaStreamDestroy(io->load_q);
  if (io->store_q) cudaStreamDestroy(io->store_q);
  delete io;
  return KVX_OK;
}

void* kvx_layer_io_load_stream(kvx_layer_io* io) { return io ? io->load_q : nullptr; }
void* kvx_layer_io_store_stream(kvx_layer_io* io) { return io ? io->store_q : nullptr; }

int kvx_layer_load_launch(kvx_layer_io* io, const kvx_pool* host, const int32_t* d_host_table,
                          kvx_pool* dev, const int32_t* d_dev_table, int64_t n, int32_t layer_lo,
                          int32_t layer_hi, void* after_stream) {
  KVX_REQUIRE(io && host && dev, "kvx_layer_load_launch: NULL argument");
  KVX_REQUIRE(kvx_pool_is_host(host) && !kvx_pool_is_host(dev),
              "kvx_layer_load_launch: loads go from a host (DRAM) pool into a device pool");
  KVX_REQUIRE(kvx_pool_device(dev) == io->device, "kvx_layer_load_launch: pool on another GPU");
  KVX_REQUIRE(0 <= layer_lo && layer_lo <= layer_hi && layer_hi <= io->max_layers,
              "kvx_layer_load_launch: bad layer range");
  kvx::DeviceGuard g(io->device);
  int rc = order_after(io, io->load_q, after_stream);
  if (rc) return rc;
  for (int32_t l = layer_lo; l < layer_hi; ++l) {  // one unit per layer, in layer order
    rc = kvx_copy_paged(host, d_host_table, dev, d_dev_table, n, l, l + 1, io->load_q);
    if (rc) return rc;
    KVX_CUDA(cudaEventRecord(io->loaded[l], io->load_q));
  }
  return KVX_OK;
}

int kvx_layer_load_wait(kvx_layer_io* io, int32_t layer, void* stream) {
  KVX_REQUIRE(io && layer >= 0 && layer < io->max_layers, "kvx_layer_load_wait: bad layer");
  kvx::DeviceGuard g(io->device);
  KVX_CUDA(cudaStreamWaitEvent(as_stream(stream), io->loaded[layer], 0));
  return KVX_OK;
}

int kvx_layer_store_launch(kvx_layer_io* io, const kvx_pool* dev, const int32_t* d_dev_table,
                           kvx_pool* host, const int32_t* d_host_table, int64_t n, int32_t layer_lo,
                           int32_t layer_hi, void* after_stream) {
  KVX_REQUIRE(io && host && dev, "kvx_layer_store_launch: NULL argument");
  KVX_REQUIRE(kvx_pool_is_host(host) && !kvx_pool_is_host(dev),
              "kvx_layer_store_launch: stores go from a device pool into a host (DRAM) pool");
  KVX_REQUIRE(kvx_pool_device(dev) == io->device, "kvx_layer_store_launch: pool on another GPU");
  KVX_REQUIRE(0 <= layer_lo && layer_lo <= layer_hi && layer_hi <= io->max_layers,
              "kvx_layer_store_launch: bad layer range");
  kvx::DeviceGuard g(io->device);
  int rc = order_after(io, io->store_q, after_stream);
  if (rc) return rc;
  for (int32_t l = layer_lo; l < layer_hi; ++l) {
    rc = kvx_copy_paged(dev, d_dev_table, host, d_host_table, n, l, l + 1, io->store_q);
    if (rc) return rc;
  }
  return KVX_OK;
}

// Contiguous runs (the block range [h0, h0+n) of the DRAM pool <-> [d0, d0+n)
// of the HBM pool): each (layer, K|V) plane is then ONE contiguous range on
// both sides, so a layer is two copy-engine copies and no kernel -- the SMs
// stay entirely with the prefill compute, which register-heavy GEMMs would
// not leave to a copy kernel anyway.
namespace {
int range_copy(kvx_layer_io* io, cudaStream_t q, const kvx_pool* from, int64_t f0, kvx_pool* to,
               int64_t t0, int64_t n, int32_t l) {
  const int64_t slab = kvx_pool_slab_bytes(from);
  const int64_t fslots = kvx_pool_bytes(from) / (2 * kvx_pool_layers(from) * slab);
  const int64_t tslots = kvx_pool_bytes(to) / (2 * kvx_pool_layers(to) * slab);
  KVX_REQUIRE(f0 >= 0 && t0 >= 0 && n >= 0 && f0 + n <= fslots && t0 + n <= tslots,
              "kvx_layer_*_range: block range outside a pool");
  auto* fb = static_cast<const uint8_t*>(kvx_pool_base(from));
  auto* tb = static_cast<uint8_t*>(kvx_pool_base(to));
  for (int kv = 0; kv < 2; ++kv) {
    const int64_t fp = ((static_cast<int64_t>(l) * 2 + kv) * fslots + f0) * slab;
    const int64_t tp = ((static_cast<int64_t>(l) * 2 + kv) * tslots + t0) * slab;
    if (n) KVX_CUDA(cudaMemcpyAsync(tb + tp, fb + fp, static_cast<size_t>(n * slab),
                                    cudaMemcpyDefault, q));
  }
  return KVX_OK;
}
}  // namespace

int kvx_layer_load_range(kvx_layer_io* io, const kvx_pool* host, int64_t host_first,
                         kvx_pool* dev, int64_t dev_first, int64_t n, int32_t layer_lo,
                         int32_t layer_hi, void* after_stream) {
  KVX_REQUIRE(io && host && dev, "kvx_layer_load_range: NULL argument");
  KVX_REQUIRE(kvx_pool_is_host(host) && !kvx_pool_is_host(dev),
              "kvx_layer_load_range: loads go from a host (DRAM) pool into a device pool");
  KVX_REQUIRE(kvx_pool_slab_bytes(host) == kvx_pool_slab_bytes(dev),
              "kvx_layer_load_range: pools have different block shapes");
  KVX_REQUIRE(0 <= layer_lo && layer_lo <= layer_hi && layer_hi <= io->max_layers &&
                  layer_hi <= kvx_pool_layers(host) && layer_hi <= kvx_pool_layers(dev),
              "kvx_layer_load_range: bad layer range");
  kvx::DeviceGuard g(io->device);
  int rc = order_after(io, io->load_q, after_stream);
  if (rc) return rc;
  for (int32_t l = layer_lo; l < layer_hi; ++l) {
    rc = range_copy(io, io->load_q, host, host_first, dev, dev_first, n, l);
    if (rc) return rc;
    KVX_CUDA(cudaEventRecord(io->loaded[l], io->load_q));
  }
  return KVX_OK;
}

int kvx_layer_store_range(kvx_layer_io* io, const kvx_pool* dev, int64_t dev_first,
                          kvx_pool* host, int64_t host_first, int64_t n, int32_t layer_lo,
                          int32_t layer_hi, void* after_stream) {
  KVX_REQUIRE(io && host && dev, "kvx_layer_store_range: NULL argument");
  KVX_REQUIRE(kvx_pool_is_host(host) && !kvx_pool_is_host(dev),
              "kvx_layer_store_range: stores go from a device pool into a host (DRAM) pool");
  KVX_REQUIRE(kvx_pool_slab_bytes(host) == kvx_pool_slab_bytes(dev),
              "kvx_layer_store_range: pools have different block shapes");
  KVX_REQUIRE(0 <= layer_lo && layer_lo <= layer_hi && layer_hi <= io->max_layers &&
                  layer_hi <= kvx_pool_layers(host) && layer_hi <= kvx_pool_layers(dev),
              "kvx_layer_store_range: bad layer range");
  kvx::DeviceGuard g(io->device);
  int rc = order_after(io, io->store_q, after_stream);
  if (rc) return rc;
  for (int32_t l = layer_lo; l < layer_hi; ++l) {
    rc = range_copy(io, io->store_q, dev, dev_first, host, host_first, n, l);
    if (rc) return rc;
  }
  return KVX_OK;
}

int kvx_layer_store_wait_all(kvx_layer_io* io, void* stream) {
  KVX_REQUIRE(io != nullptr, "kvx_layer_store_wait_all: NULL");
  kvx::DeviceGuard g(io->device);
  KVX_CUDA(cudaEventRecord(io->stored, io->store_q));
  if (stream) {
    KVX_CUDA(cudaStreamWaitEvent(as_stream(stream), io->stored, 0));
  } else {
    KVX_CUDA(cudaEventSynchronize(io->stored));
  }
  return KVX_OK;
}

}  // extern "C"
