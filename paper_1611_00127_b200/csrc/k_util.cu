// k_util.cu -- prefix scans and the stable key/value radix sort used by the
// deterministic setup (CUB device primitives, the one library dependency of the
// setup path: a scan and a sort are library steps, the method's arithmetic is ours).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "bf_internal.cuh"
BF_CHECK_TU("k_util.cu")

namespace bf {

// input of the scans: counts[0..n) followed by one zero, without a padded copy
template <typename T>
struct PaddedCounts {
  const T *p;
  int64_t n;
  __host__ __device__ T operator()(int64_t i) const { return i < n ? p[i] : T(0); }
};
template <typename T>
static auto padded_input(const T *counts, int64_t n) {
  return thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), PaddedCounts<T>{counts, n});
}

int64_t exclusive_scan_i32(bf_ctx *c, const int32_t *counts, int32_t *out, int32_t n) {
  // out[0..n] with out[n] = total; the total must fit int32 (checked by the caller's allocator)
  size_t tmp = 0;
  auto in = padded_input(counts, n);
  BF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1, c->stream));
  void *t = dalloc(c, tmp + 16);
  BF_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n + 1, c->stream));
  c->launches += 2;
  int32_t total = 0;
  BF_CUDA(cudaMemcpyAsync(&total, out + n, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, t);
  return total;
}

int64_t exclusive_scan_i64(bf_ctx *c, const int64_t *counts, int64_t *out, int64_t n) {
  size_t tmp = 0;
  auto in = padded_input(counts, n);
  BF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1, c->stream));
  void *t = dalloc(c, tmp + 16);
  BF_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n + 1, c->stream));
  c->launches += 2;
  int64_t total = 0;
  BF_CUDA(cudaMemcpyAsync(&total, out + n, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, t);
  return total;
}

// stable LSD radix sort of (key, value) pairs by the low end_bit bits of the key (in place)
void sort_pairs_u64_f64(bf_ctx *c, uint64_t *keys, double *vals, int64_t count, int end_bit) {
  if (count <= 1) return;
  uint64_t *k2 = dalloc_t<uint64_t>(c, count);
  double *v2 = dalloc_t<double>(c, count);
  cub::DoubleBuffer<uint64_t> kb(keys, k2);
  cub::DoubleBuffer<double> vb(vals, v2);
  size_t tmp = 0;
  BF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, count, 0, end_bit, c->stream));
  void *t = dalloc(c, tmp + 16);
  BF_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, count, 0, end_bit, c->stream));
  c->launches += 4;
  if (kb.Current() != keys) {
    BF_CUDA(cudaMemcpyAsync(keys, kb.Current(), sizeof(uint64_t) * count, cudaMemcpyDeviceToDevice, c->stream));
    BF_CUDA(cudaMemcpyAsync(vals, vb.Current(), sizeof(double) * count, cudaMemcpyDeviceToDevice, c->stream));
  }
  dfree(c, t);
  dfree(c, k2);
  dfree(c, v2);
}

// stable radix sort of (key, int32 value) pairs by the low end_bit bits of the key (in place)
void sort_pairs_u64_i32(bf_ctx *c, uint64_t *keys, int32_t *vals, int64_t count, int end_bit) {
  if (count <= 1) return;
  uint64_t *k2 = dalloc_t<uint64_t>(c, count);
  int32_t *v2 = dalloc_t<int32_t>(c, count);
  cub::DoubleBuffer<uint64_t> kb(keys, k2);
  cub::DoubleBuffer<int32_t> vb(vals, v2);
  size_t tmp = 0;
  BF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, count, 0, end_bit, c->stream));
  void *t = dalloc(c, tmp + 16);
  BF_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, count, 0, end_bit, c->stream));
  c->launches += 4;
  if (kb.Current() != keys) {
    BF_CUDA(cudaMemcpyAsync(keys, kb.Current(), sizeof(uint64_t) * count, cudaMemcpyDeviceToDevice, c->stream));
    BF_CUDA(cudaMemcpyAsync(vals, vb.Current(), sizeof(int32_t) * count, cudaMemcpyDeviceToDevice, c->stream));
  }
  dfree(c, t);
  dfree(c, k2);
  dfree(c, v2);
}

}  // namespace bf
