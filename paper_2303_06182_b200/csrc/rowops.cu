// Bandwidth-bound row kernels around the grouped FFN:
//   gather   Xp[p] = X[order[p] / k]  (zero row for static placeholders)
//            -- the paper's O(S*D) "indexing operation",
//               counted by the reference as gather_elements = k*S*TD
//               (proj/src/gating.cpp:123)
//   combine  out[t] = sum_j Yw[pos[t*k+j]]  (gate weights were applied in the
//            GEMM2 epilogue; dropped slots, pos = -1, contribute nothing)
//            -- the weighted form of combine<T> (proj/include/moesim/
//               gating.hpp:107-184): each token gathers its k expert outputs
//               in assignment-slot order (j = 0..k-1), so the fp32 sum order
//               is fixed and the result is deterministic.
//   fill     counter-based synthetic data (bit-identical to oracle/layer.py)
// One warp per row, 16-byte vector accesses, 4 independent loads in flight
// per lane.
#include "moe_internal.h"
#include "ptx.cuh"

namespace moe {

namespace {

__global__ void __launch_bounds__(256)
    gather_rows_kernel(const uint4* __restrict__ X, const int32_t* __restrict__ order, int rows,
                       int k, int vec_per_row, uint4* __restrict__ Xp, int late) {
  if (!late) pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int p = warp; p < rows; p += nwarps) {
    const int slot = order[p];
    uint4* dst = Xp + static_cast<size_t>(p) * vec_per_row;
    if (slot < 0) {
      for (int v = lane; v < vec_per_row; v += 32) dst[v] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint4* src = X + static_cast<size_t>(slot / k) * vec_per_row;
    int v = lane;
    for (; v + 96 < vec_per_row; v += 128) {
      const uint4 a = __ldg(src + v), b = __ldg(src + v + 32), c = __ldg(src + v + 64),
                  d = __ldg(src + v + 96);
      dst[v] = a;
      dst[v + 32] = b;
      dst[v + 64] = c;
      dst[v + 96] = d;
    }
    for (; v < vec_per_row; v += 32) dst[v] = __ldg(src + v);
  }
  if (late) pdl_trigger();
}

__device__ __forceinline__ void add_bf16x8(float (&acc)[8], const uint4& v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    acc[2 * i] += f.x;
    acc[2 * i + 1] += f.y;
  }
}

__global__ void __launch_bounds__(256)
    combine_kernel(const uint4* __restrict__ Yw, const int32_t* __restrict__ pos, int S, int k,
                   int vec_per_row, uint4* __restrict__ out, int late) {
  if (!late) pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < S; t += nwarps) {
    for (int v = lane; v < vec_per_row; v += 32) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < k; ++j) {
        const int p = pos[static_cast<size_t>(t) * k + j];
        if (p >= 0) add_bf16x8(acc, __ldg(Yw + static_cast<size_t>(p) * vec_per_row + v));
      }
      uint4 o;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      out[static_cast<size_t>(t) * vec_per_row + v] = o;
    }
  }
  if (late) pdl_trigger();
}

// Same arithmetic as combine_kernel for a compile-time k: the token's k slot
// rows are read once, then each lane keeps 4 x k independent 16-byte loads in
// flight (the generic loop has k, behind a dependent pos load).  Sums stay in
// slot order, dropped slots (pos < 0) are skipped: bitwise equal.
template <int K>
__global__ void __launch_bounds__(256)
    combine_k_kernel(const uint4* __restrict__ Yw, const int32_t* __restrict__ pos, int S,
                     int vec_per_row, uint4* __restrict__ out, int late) {
  if (!late) pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < S; t += nwarps) {
    const uint4* src[K];
    bool live[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int p = pos[static_cast<size_t>(t) * K + j];
      live[j] = p >= 0;
      src[j] = Yw + static_cast<size_t>(live[j] ? p : 0) * vec_per_row;
    }
    uint4* dst = out + static_cast<size_t>(t) * vec_per_row;
    int v = lane;
    for (; v + 96 < vec_per_row; v += 128) {
      uint4 x[K][4];
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (live[j]) x[j][u] = __ldg(src[j] + v + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (live[j]) add_bf16x8(acc, x[j][u]);
        uint4 o;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
        dst[v + 32 * u] = o;
      }
    }
    for (; v < vec_per_row; v += 32) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (live[j]) add_bf16x8(acc, __ldg(src[j] + v));
      uint4 o;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      dst[v] = o;
    }
  }
  if (late) pdl_trigger();
}

// Gather by token (dynamic gating: pos is a bijection slot -> row, no
// placeholder rows): each X row is read once and stored to its k expert rows,
// 4 loads and 4k stores in flight per lane -- X is read once instead of k
// times (the row form relies on L2 for the repeats).
template <int K>
__global__ void __launch_bounds__(256)
    gather_tokens_k_kernel(const uint4* __restrict__ X, const int32_t* __restrict__ pos, int S,
                           int vec_per_row, uint4* __restrict__ Xp, int late) {
  if (!late) pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < S; t += nwarps) {
    uint4* dst[K];
    bool live[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int p = pos[static_cast<size_t>(t) * K + j];
      live[j] = p >= 0;
      dst[j] = Xp + static_cast<size_t>(live[j] ? p : 0) * vec_per_row;
    }
    const uint4* src = X + static_cast<size_t>(t) * vec_per_row;
    int v = lane;
    for (; v + 96 < vec_per_row; v += 128) {
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldg(src + v + 32 * u);
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (live[j]) dst[j][v + 32 * u] = x[u];
    }
    for (; v < vec_per_row; v += 32) {
      const uint4 x = __ldg(src + v);
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (live[j]) dst[j][v] = x;
    }
  }
  if (late) pdl_trigger();
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// value(i) = (int(h >> 40) - 2^23) * 2^-23 * scale, h = mix64(seed*phi +
// tensor_id*c + i): uniform on [-scale, scale), exactly reproducible on the
// CPU (oracle/layer.py::synth) because every step is an exact integer op or a
// single IEEE fp32 rounding.
__global__ void fill_uniform_bf16_kernel(__nv_bfloat16* dst, int64_t n, uint64_t seed,
                                         uint64_t tensor_id, float scale) {
  const uint64_t base = seed * 0x9E3779B97F4A7C15ull + tensor_id * 0xD1B54A32D192ED03ull;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(base + static_cast<uint64_t>(i));
    const int32_t u = static_cast<int32_t>(h >> 40) - (1 << 23);
    const float x = __fmul_rn(static_cast<float>(u) * 0x1p-23f, scale);
    dst[i] = __float2bfloat16_rn(x);
  }
}

// out[r] = (segment of r) % mod, segments laid out back to back with the
// given lengths (one warp per segment).
__global__ void fill_segments_kernel(const int32_t* __restrict__ counts, int n, int mod,
                                     int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  // exclusive offsets recomputed per segment: n is small (D * E_local)
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < n; s += nwarps) {
    int off = 0;
    for (int i = lane; i < s; i += 32) off += counts[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
    const int len = counts[s];
    for (int r = lane; r < len; r += 32) out[off + r] = s % mod;
  }
}

// Release the next kernel of the chain only when this one's CTAs finish
// instead of at their start (see ffn_fused.cu).  Default on for the combine
// (the next step's gate CTAs, 200 KB of smem each, otherwise sit resident
// while it streams: 8-25 us per LM step, 3 of 3 same-box A/B rounds), off for
// the gather (no consistent effect).
int late_trigger(const char* env, int dflt) {
  const char* v = getenv(env);
  return v ? atoi(v) : dflt;
}

int grid_for(int64_t warps_needed, int sms) {
  const int64_t blocks = (warps_needed + 7) / 8;
  const int64_t cap = static_cast<int64_t>(sms) * 16;
  return static_cast<int>(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

}  // namespace

cudaError_t launch_gather_rows(const __nv_bfloat16* X, const int32_t* order, int rows, int k,
                               int TD, __nv_bfloat16* Xp, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  return launch_chain(gather_rows_kernel, dim3(grid_for(rows, sm_count())), dim3(256), 0, stream,
                      false, reinterpret_cast<const uint4*>(X), order, rows, k, TD / 8,
                      reinterpret_cast<uint4*>(Xp), late_trigger("MOE_GATHER_LATE_TRIGGER", 0));
}

cudaError_t launch_gather_tokens(const __nv_bfloat16* X, const int32_t* pos, int S, int k,
                                 int TD, __nv_bfloat16* Xp, cudaStream_t stream) {
  if (S <= 0) return cudaSuccess;
  const int late = late_trigger("MOE_GATHER_LATE_TRIGGER", 0);
  const dim3 grid(grid_for(S, sm_count()));
  const uint4* x = reinterpret_cast<const uint4*>(X);
  uint4* xp = reinterpret_cast<uint4*>(Xp);
  switch (k) {
    case 1: return launch_chain(gather_tokens_k_kernel<1>, grid, dim3(256), 0, stream, false, x, pos, S, TD / 8, xp, late);
    case 2: return launch_chain(gather_tokens_k_kernel<2>, grid, dim3(256), 0, stream, false, x, pos, S, TD / 8, xp, late);
    case 3: return launch_chain(gather_tokens_k_kernel<3>, grid, dim3(256), 0, stream, false, x, pos, S, TD / 8, xp, late);
    case 4: return launch_chain(gather_tokens_k_kernel<4>, grid, dim3(256), 0, stream, false, x, pos, S, TD / 8, xp, late);
    default: return cudaErrorInvalidValue;
  }
}

bool gather_by_token(int k) {
  static const int env = [] {
    const char* v = getenv("MOE_GATHER_TOKENS");
    return v ? atoi(v) : 1;
  }();
  return env != 0 && k >= 1 && k <= 4;
}

cudaError_t launch_combine(const __nv_bfloat16* Yw, const int32_t* pos, int S, int k, int TD,
                           __nv_bfloat16* out, cudaStream_t stream) {
  if (S <= 0) return cudaSuccess;
  const int late = late_trigger("MOE_COMBINE_LATE_TRIGGER", 1);
  static const bool by_k = [] {
    const char* e = getenv("MOE_COMBINE_K");
    return e ? atoi(e) != 0 : true;
  }();
  const dim3 grid(grid_for(S, sm_count()));
  const uint4* y = reinterpret_cast<const uint4*>(Yw);
  uint4* o = reinterpret_cast<uint4*>(out);
  if (by_k) {
    switch (k) {
      case 1: return launch_chain(combine_k_kernel<1>, grid, dim3(256), 0, stream, false, y, pos, S, TD / 8, o, late);
      case 2: return launch_chain(combine_k_kernel<2>, grid, dim3(256), 0, stream, false, y, pos, S, TD / 8, o, late);
      case 3: return launch_chain(combine_k_kernel<3>, grid, dim3(256), 0, stream, false, y, pos, S, TD / 8, o, late);
      case 4: return launch_chain(combine_k_kernel<4>, grid, dim3(256), 0, stream, false, y, pos, S, TD / 8, o, late);
      default: break;
    }
  }
  return launch_chain(combine_kernel, grid, dim3(256), 0, stream, false, y, pos, S, k, TD / 8, o,
                      late);
}

cudaError_t launch_fill_segments(const int32_t* counts, int n_segments, int mod, int32_t* out,
                                 cudaStream_t stream) {
  if (n_segments <= 0) return cudaSuccess;
  fill_segments_kernel<<<grid_for(n_segments, sm_count()), 256, 0, stream>>>(counts, n_segments,
                                                                             mod, out);
  return cudaGetLastError();
}

cudaError_t launch_fill_uniform_bf16(__nv_bfloat16* dst, int64_t n, uint64_t seed,
                                     uint64_t tensor_id, float scale, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  fill_uniform_bf16_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(dst, n, seed, tensor_id,
                                                                          scale);
  return cudaGetLastError();
}

// Weight prepack: row-major [mblocks * 128, K] -> tiles of 128 rows x 64
// columns, each 16 KB contiguous, tile (mb, kc) at tile index mb * (K/64) + kc,
// rows 128 B apart with the 128-byte swizzle already applied.
// One CTA per tile: 128 rows x 8 x 16 B.
__global__ void pack_tiles_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int K) {
  const long tile = blockIdx.x;
  const int kc_n = K / 64;
  const long mb = tile / kc_n;
  const int kc = static_cast<int>(tile % kc_n);
  const int vrow = K / 8;  // uint4 per source row
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    // 16-byte chunk c of row r at chunk c ^ (r % 8): the 128-byte swizzle the
    // UMMA descriptors expect, applied here once instead of by every TMA load
    dst[tile * 1024 + r * 8 + (c ^ (r & 7))] = src[(mb * 128 + r) * vrow + kc * 8 + c];
  }
}

cudaError_t launch_pack_tiles(const __nv_bfloat16* src, __nv_bfloat16* dst, long rows, int K,
                              cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (rows % 128 || K % 64) return cudaErrorInvalidValue;
  const long tiles = rows / 128 * (K / 64);
  if (tiles > 0x7fffffffL) return cudaErrorInvalidValue;
  pack_tiles_kernel<<<static_cast<unsigned>(tiles), 256, 0, stream>>>(
      reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), K);
  return cudaGetLastError();
}

}  // namespace moe
