// segment.cu — S0: world segmentation of the contact set (integer, bit-exact).
//
// The contact set C arrives as a list with a world id per
// contact.  The step kernel needs the contacts of each world contiguous and
// their CSR offsets off[W+1]; impulse outputs need per-contact facet offsets
// foff[n+1] (facet sets of Eq. (7)-(8)).
//   sorted input   : one pass detects world boundaries and writes off[],
//                    verifying the promised order (4 B/contact read).
//   unsorted input : stable radix sort of (world, index) pairs (CUB), then
//                    boundaries on the sorted keys and a gather of the four
//                    contact streams into library scratch.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.h"

namespace cf {

// off[k] = first position whose world id >= k, for k in [0, W]; every entry is
// written exactly once when the ids are non-decreasing.  Each thread scans 8
// consecutive ids (two 128-bit loads when aligned) so the 4 B/contact read is
// issued by one wave of threads.
__device__ __forceinline__ void boundary(int64_t c, int64_t prev, int64_t cur, int64_t n, int64_t W,
                                         int64_t* __restrict__ off, int* err) {
  if (c < n && (cur < 0 || cur >= W)) {
    atomicOr(err, ERR_WORLD_RANGE);
    return;
  }
  if (cur < prev) {
    atomicOr(err, ERR_UNSORTED);
    return;
  }
  if (prev < -1) prev = -1;
  for (int64_t k = prev + 1; k <= cur && k <= W; ++k) off[k] = c;
}

__global__ void k_offsets_sorted(const int32_t* __restrict__ world, int64_t n, int64_t W,
                                 int64_t* __restrict__ off, int* err) {
  const int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c0 > n) return;
  int32_t v[8];
  const bool aligned = ((reinterpret_cast<uintptr_t>(world) & 15) == 0);
  if (aligned && c0 + 8 <= n) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(world + c0));
    const int4 b = __ldg(reinterpret_cast<const int4*>(world + c0 + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (c0 + j < n) ? __ldg(world + c0 + j) : (int32_t)W;
  }
  int64_t prev = (c0 == 0) ? -1 : (int64_t)__ldg(world + c0 - 1);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t c = c0 + j;
    if (c > n) break;
    const int64_t cur = (c == n) ? W : (int64_t)v[j];
    if (cur != prev || c == n) boundary(c, prev, cur, n, W, off, err);
    prev = cur;
  }
}

__global__ void k_check_range(const int32_t* __restrict__ world, int64_t n, int64_t W, int* err) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n && (world[c] < 0 || world[c] >= W)) atomicOr(err, ERR_WORLD_RANGE);
}

__global__ void k_iota(int32_t* out, int64_t n) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) out[c] = (int32_t)c;
}

__global__ void k_gather(const int32_t* __restrict__ perm, int64_t n, const float4* __restrict__ c0,
                         const float4* __restrict__ c1, const float4* __restrict__ c2,
                         const int4* __restrict__ c3, const float4* __restrict__ jrow,
                         const float2* __restrict__ kd,
                         float4* __restrict__ o0, float4* __restrict__ o1, float4* __restrict__ o2,
                         int4* __restrict__ o3, float4* __restrict__ oj, float2* __restrict__ okd) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t src = perm[i];
  o0[i] = c0[src];
  o1[i] = c1[src];
  o2[i] = c2[src];
  o3[i] = c3[src];
  if (jrow)
    for (int s = 0; s < 12; ++s) oj[(size_t)s * n + i] = jrow[(size_t)s * n + src];
  if (kd) okd[i] = kd[src];
}

// facets per contact (condim -> 1 / n_t / n_t + 2 / n_t + 2 + n_rol); the
// trailing element is 0 so the exclusive scan of n + 1 values ends in F.
__global__ void k_nfacets(const int4* __restrict__ c3, int64_t n, int n_t, int n_rol,
                          int32_t* __restrict__ nf, int* err) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n) return;
  if (c == n) { nf[c] = 0; return; }
  const int cd = c3[c].w;
  int v;
  switch (cd) {
    case 1: v = 1; break;
    case 3: v = n_t; break;
    case 4: v = n_t + 2; break;
    case 6: v = n_t + 2 + n_rol; break;
    default: v = 0; atomicOr(err, ERR_CONDIM);
  }
  nf[c] = v;
}

static unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_offsets_sorted(const int32_t* world, int64_t n, int64_t W, int64_t* off, int* err,
                                  cudaStream_t s) {
  k_offsets_sorted<<<blocks_for((n + 1 + 7) / 8), 256, 0, s>>>(world, n, W, off, err);
  return cudaGetLastError();
}

cudaError_t launch_check_world_range(const int32_t* world, int64_t n, int64_t W, int* err, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_check_range<<<blocks_for(n), 256, 0, s>>>(world, n, W, err);
  return cudaGetLastError();
}

cudaError_t launch_iota(int32_t* out, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_iota<<<blocks_for(n), 256, 0, s>>>(out, n);
  return cudaGetLastError();
}

static int bits_for(int64_t W) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) < W) ++b;
  return b;
}

// Stable (world, index) sort.  temp == nullptr queries *temp_bytes.
cudaError_t sort_by_world(const int32_t* world, int64_t n, int64_t W, int32_t* keys_out, int32_t* perm_out,
                          int32_t* iota_tmp, void* temp, size_t* temp_bytes, cudaStream_t s) {
  return cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, world, keys_out, iota_tmp, perm_out, (int)n, 0,
                                         bits_for(W + 1), s);
}

cudaError_t launch_gather_contacts(const int32_t* perm, int64_t n, const float4* c0, const float4* c1,
                                   const float4* c2, const int4* c3, const float4* jrow, const float2* kd,
                                   float4* o0, float4* o1, float4* o2, int4* o3, float4* oj, float2* okd,
                                   cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_gather<<<blocks_for(n), 256, 0, s>>>(perm, n, c0, c1, c2, c3, jrow, kd, o0, o1, o2, o3, oj, okd);
  return cudaGetLastError();
}

// foff[n+1] = exclusive prefix of facets per contact (input order).  temp ==
// nullptr queries *temp_bytes (nf_tmp may be null then).
cudaError_t facet_offsets(const int4* c3, int64_t n, int n_t, int n_rol, int32_t* nf_tmp, int64_t* foff,
                          void* temp, size_t* temp_bytes, int* err, cudaStream_t s) {
  if (temp == nullptr)
    return cub::DeviceScan::ExclusiveSum(nullptr, *temp_bytes, (const int32_t*)nullptr, (int64_t*)nullptr,
                                         (int)(n + 1), s);
  k_nfacets<<<blocks_for(n + 1), 256, 0, s>>>(c3, n, n_t, n_rol, nf_tmp, err);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, (const int32_t*)nf_tmp, foff, (int)(n + 1), s);
}

}  // namespace cf
