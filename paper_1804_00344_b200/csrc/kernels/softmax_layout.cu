// Masked softmax (softmaxInto tensor.cpp:393-440, graph.cpp:526-555) and the
// layout kernels: transposeInto / concatInto / sliceInto (tensor.cpp:480-541),
// gatherRowsInto / scatterAddRows (:456-476) and the embedding lookup fused
// with the positional encoding (graph.cpp:595-622 + layers.cpp:164-179).
#include <algorithm>

#include "common.cuh"

using namespace mtkc;

namespace {

struct SmP {
  float* out;
  const float* x;
  const float* mask;
  int64_t rows, cols;
  int64_t xd[4];
  int64_t ms[4];
  int logMode;
  int* flags;
};

// One warp per row.  Two passes over the row like the reference: max over
// unmasked entries, then sum of exp(x - max) over unmasked entries.
__global__ void softmax_kernel(SmP p) {
  MTKC_PDL_ENTRY();
  int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if(row >= p.rows)
    return;
  const float* xr = p.x + row * p.cols;
  float* orow = p.out + row * p.cols;
  int64_t moff = 0;
  if(p.mask) {
    int64_t i2 = row % p.xd[2], rest = row / p.xd[2];
    int64_t i1 = rest % p.xd[1], i0 = rest / p.xd[1];
    moff = i0 * p.ms[0] + i1 * p.ms[1] + i2 * p.ms[2];
  }
  auto m = [&](int64_t j) -> bool { return !p.mask || p.mask[moff + j * p.ms[3]] != 0.f; };
  float mx = -INFINITY;
  int any = 0;
  for(int64_t j = lane; j < p.cols; j += 32)
    if(m(j)) {
      any = 1;
      mx = fmaxf(mx, xr[j]);
    }
  mx = warp_max(mx);
  any = __any_sync(0xffffffffu, any);
  if(!any) {
    if(lane == 0 && p.flags)
      atomicOr(p.flags, MTKC_FLAG_MASKED_ROW);
    for(int64_t j = lane; j < p.cols; j += 32)
      orow[j] = p.logMode ? -INFINITY : 0.f;
    return;
  }
  float s = 0.f;
  for(int64_t j = lane; j < p.cols; j += 32)
    if(m(j))
      s += expf(xr[j] - mx);
  s = warp_sum(s);
  if(p.logMode) {
    float lz = mx + logf(s);
    for(int64_t j = lane; j < p.cols; j += 32)
      orow[j] = m(j) ? xr[j] - lz : -INFINITY;
  } else {
    for(int64_t j = lane; j < p.cols; j += 32)
      orow[j] = m(j) ? expf(xr[j] - mx) / s : 0.f;
  }
}

// dx += y * (g - sum(g*y))  (graph.cpp:539-552)
__global__ void softmax_bwd_kernel(float* gx, const float* y, const float* go, int64_t rows,
                                   int64_t cols) {
  MTKC_PDL_ENTRY();
  int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if(row >= rows)
    return;
  const float* yr = y + row * cols;
  const float* gr = go + row * cols;
  float* xr = gx + row * cols;
  float d = 0.f;
  for(int64_t j = lane; j < cols; j += 32)
    d += gr[j] * yr[j];
  d = warp_sum(d);
  for(int64_t j = lane; j < cols; j += 32)
    xr[j] += yr[j] * (gr[j] - d);
}

struct TrP {
  float* out;
  const float* src;
  int64_t od[4];
  int64_t ss[4];  // source stride for each output dim
  int64_t n;
  int acc;
};

__global__ void transpose_kernel(TrP p) {
  MTKC_PDL_ENTRY();
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int64_t i3 = r % p.od[3];
    r /= p.od[3];
    int64_t i2 = r % p.od[2];
    r /= p.od[2];
    int64_t i1 = r % p.od[1];
    int64_t i0 = r / p.od[1];
    float v = p.src[i0 * p.ss[0] + i1 * p.ss[1] + i2 * p.ss[2] + i3 * p.ss[3]];
    p.out[i] = p.acc ? p.out[i] + v : v;
  }
}

// float4 form when the innermost output dim is contiguous in the source (a
// permutation of row blocks, e.g. batch-major <-> time-major activations):
// one index decomposition per 4 elements, 32-bit when the sizes allow
template <typename I>
__global__ void transpose4_kernel(TrP p) {
  MTKC_PDL_ENTRY();
  const I n4 = (I)(p.n / 4), d3 = (I)(p.od[3] / 4), d2 = (I)p.od[2], d1 = (I)p.od[1];
  float4* out4 = reinterpret_cast<float4*>(p.out);
  for(I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < n4; i += (I)gridDim.x * blockDim.x) {
    I r = i;
    const I c4 = r % d3;
    r /= d3;
    const I i2 = r % d2;
    r /= d2;
    const I i1 = r % d1;
    const I i0 = r / d1;
    const float4 v = *reinterpret_cast<const float4*>(
        p.src + (int64_t)i0 * p.ss[0] + (int64_t)i1 * p.ss[1] + (int64_t)i2 * p.ss[2] +
        4 * (int64_t)c4);
    if(p.acc) {
      const float4 o = out4[i];
      out4[i] = make_float4(o.x + v.x, o.y + v.y, o.z + v.z, o.w + v.w);
    } else {
      out4[i] = v;
    }
  }
}

template <typename I>
__global__ void copy_blocks4_kernel(float* dst, int64_t dstStride, int64_t dstOff,
                                    const float* src, int64_t srcStride, int64_t srcOff,
                                    int64_t outer, int64_t len, int acc) {
  MTKC_PDL_ENTRY();
  const I l4 = (I)(len / 4), n4 = (I)(outer * (len / 4));
  for(I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < n4; i += (I)gridDim.x * blockDim.x) {
    const I o = i / l4, j = i - o * l4;
    const float4 v =
        *reinterpret_cast<const float4*>(src + (int64_t)o * srcStride + srcOff + 4 * (int64_t)j);
    float4* d = reinterpret_cast<float4*>(dst + (int64_t)o * dstStride + dstOff + 4 * (int64_t)j);
    if(acc) {
      const float4 x = *d;
      *d = make_float4(x.x + v.x, x.y + v.y, x.z + v.z, x.w + v.w);
    } else {
      *d = v;
    }
  }
}

struct CopyJobs {
  mtkc_copy_job j[MTKC_COPY_MAX_JOBS];
  int n;
};

// several strided 2-d copies in one launch (blockIdx.y = job)
__global__ void copy_many_kernel(const __grid_constant__ CopyJobs cj) {
  MTKC_PDL_ENTRY();
  const mtkc_copy_job& J = cj.j[blockIdx.y];
  const int64_t n = J.rows * J.cols;
  if(J.cols % 4 == 0 && J.lds % 4 == 0 && J.ldd % 4 == 0 &&
     (((uintptr_t)J.src | (uintptr_t)J.dst) & 15) == 0) {  // float4 rows
    const int64_t c4 = J.cols / 4, n4 = J.rows * c4;
    for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
        i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / c4, c = (i - r * c4) * 4;
      float4 v = *reinterpret_cast<const float4*>(J.src + r * J.lds + c);
      float4* d = reinterpret_cast<float4*>(J.dst + r * J.ldd + c);
      if(J.accumulate) {
        const float4 o = *d;
        v = make_float4(o.x + v.x, o.y + v.y, o.z + v.z, o.w + v.w);
      }
      *d = v;
    }
    return;
  }
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / J.cols, c = i - r * J.cols;
    const float v = J.src[r * J.lds + c];
    float* d = J.dst + r * J.ldd + c;
    *d = J.accumulate ? *d + v : v;
  }
}

__global__ void copy_blocks_kernel(float* dst, int64_t dstStride, int64_t dstOff,
                                   const float* src, int64_t srcStride, int64_t srcOff,
                                   int64_t outer, int64_t len, int acc) {
  MTKC_PDL_ENTRY();
  int64_t n = outer * len;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = i / len, j = i % len;
    float v = src[o * srcStride + srcOff + j];
    float* d = dst + o * dstStride + dstOff + j;
    *d = acc ? *d + v : v;
  }
}

__global__ void gather_rows_kernel(float* out, const float* src, const int32_t* rows, int64_t n,
                                   int64_t cols, int64_t srcRows, int* flags) {
  MTKC_PDL_ENTRY();
  int64_t total = n * cols;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i % cols;
    int32_t id = rows[r];
    if(id < 0 || id >= srcRows) {
      if(flags && c == 0)
        atomicOr(flags, MTKC_FLAG_BAD_ID);
      out[i] = 0.f;
      continue;
    }
    out[i] = src[(int64_t)id * cols + c];
  }
}

// One CTA per unique row id; threads stride over columns; the segment is
// summed in original position order (stable sort), starting from out[id].
__global__ void scatter_add_kernel(float* out, const float* src, const int32_t* perm,
                                   const int32_t* seg, const int32_t* uniq, int64_t cols,
                                   float scale) {
  MTKC_PDL_ENTRY();
  int64_t u = blockIdx.x;
  int64_t id = uniq[u];
  int32_t s0 = seg[u], s1 = seg[u + 1];
  float* dst = out + id * cols;
  for(int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float acc = dst[c];
    for(int32_t k = s0; k < s1; ++k) {
      float v = src[(int64_t)perm[k] * cols + c];
      acc += scale == 1.f ? v : scale * v;
    }
    dst[c] = acc;
  }
}

// Chunked scatter-add: CTA per chunk; single-chunk segments add straight
// into the table row in position order (bit-exact with the reference loop),
// chunks of long segments write partial sums.
__global__ void scatter_chunk_kernel(float* out, const float* src, const int32_t* perm,
                                     const int32_t* cstart, const int32_t* crow,
                                     const int32_t* cslot, float* partial, int64_t cols,
                                     float scale) {
  MTKC_PDL_ENTRY();
  int64_t c = blockIdx.x;
  int32_t k0 = cstart[c], k1 = cstart[c + 1];
  int32_t slot = cslot[c];
  float* dst = slot < 0 ? out + (int64_t)crow[c] * cols : partial + (int64_t)slot * cols;
  for(int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    float acc = slot < 0 ? dst[j] : 0.f;
    int32_t k = k0;
    for(; k + 4 <= k1; k += 4) {  // four independent loads in flight
      float v0 = src[(int64_t)perm[k] * cols + j], v1 = src[(int64_t)perm[k + 1] * cols + j];
      float v2 = src[(int64_t)perm[k + 2] * cols + j], v3 = src[(int64_t)perm[k + 3] * cols + j];
      if(scale != 1.f) {
        v0 *= scale;
        v1 *= scale;
        v2 *= scale;
        v3 *= scale;
      }
      acc += v0;
      acc += v1;
      acc += v2;
      acc += v3;
    }
    for(; k < k1; ++k) {
      float v = src[(int64_t)perm[k] * cols + j];
      acc += scale == 1.f ? v : scale * v;
    }
    dst[j] = acc;
  }
}

__global__ void scatter_multi_kernel(float* out, const float* partial, const int32_t* mfirst,
                                     const int32_t* mrow, int64_t cols) {
  MTKC_PDL_ENTRY();
  int64_t m = blockIdx.x;
  float* dst = out + (int64_t)mrow[m] * cols;
  for(int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    float acc = dst[j];
    for(int32_t s = mfirst[m]; s < mfirst[m + 1]; ++s)
      acc += partial[(int64_t)s * cols + j];
    dst[j] = acc;
  }
}

// out[n,:] = table[id,:]*s + pe[n % t,:]; exact gather when s == 1, pe == 0.
__global__ void embed_kernel(float* out, const float* table, const int32_t* ids, int64_t n,
                             int64_t e, int64_t vocab, float s, const float* pe, int64_t t,
                             int* flags) {
  MTKC_PDL_ENTRY();
  int64_t total = n * e;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / e, c = i % e;
    int32_t id = ids[r];
    if(id < 0 || id >= vocab) {
      if(flags && c == 0)
        atomicOr(flags, MTKC_FLAG_BAD_ID);
      out[i] = 0.f;
      continue;
    }
    float v = table[(int64_t)id * e + c];
    if(s != 1.f)
      v = s * v;
    if(pe)
      v = v + pe[(r % t) * e + c];
    out[i] = v;
  }
}

__global__ void embed4_kernel(float4* out, const float4* table, const int32_t* ids, int64_t n,
                              int64_t e4, int64_t vocab, float s, const float4* pe, int64_t t,
                              int* flags, const int32_t* pos) {
  MTKC_PDL_ENTRY();
  int64_t total = n * e4;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
      i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / e4, c = i % e4;
    int32_t id = ids[r];
    if(id < 0 || id >= vocab) {
      if(flags && c == 0)
        atomicOr(flags, MTKC_FLAG_BAD_ID);
      out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    float4 v = table[(int64_t)id * e4 + c];
    if(s != 1.f) {
      v.x = s * v.x;
      v.y = s * v.y;
      v.z = s * v.z;
      v.w = s * v.w;
    }
    if(pe) {
      float4 q = pe[(pos ? (int64_t)pos[r] : r % t) * e4 + c];
      v.x = v.x + q.x;
      v.y = v.y + q.y;
      v.z = v.z + q.z;
      v.w = v.w + q.w;
    }
    out[i] = v;
  }
}

}  // namespace

extern "C" {

int mtkc_softmax(float* out, const float* x, const int64_t xd[4], const float* mask,
                 const int64_t md[4], int log_mode, int* flags, void* stream) {
  SmP p;
  p.out = out;
  p.x = x;
  p.mask = mask;
  p.cols = xd[3];
  p.rows = xd[0] * xd[1] * xd[2];
  for(int i = 0; i < 4; ++i)
    p.xd[i] = xd[i];
  if(mask) {
    Bcast4 ms = bcast_strides(md);
    for(int i = 0; i < 4; ++i) {
      if(md[i] != 1 && md[i] != xd[i])
        return fail(MTKC_DIMENSION, "softmax: mask not broadcastable to input");
      p.ms[i] = ms.s[i];
    }
  } else {
    for(int i = 0; i < 4; ++i)
      p.ms[i] = 0;
  }
  p.logMode = log_mode;
  p.flags = flags;
  if(p.rows <= 0)
    return MTKC_OK;
  ::mtkc::launch(softmax_kernel, (unsigned)cdiv(p.rows, 8), 256, 0, S(stream), p);
  MTKC_POST_LAUNCH("softmax_kernel");
  return MTKC_OK;
}

int mtkc_softmax_backward(float* gx, const float* y, const float* go, int64_t rows,
                          int64_t cols, void* stream) {
  if(rows <= 0)
    return MTKC_OK;
  ::mtkc::launch(softmax_bwd_kernel, (unsigned)cdiv(rows, 8), 256, 0, S(stream), gx, y, go, rows, cols);
  MTKC_POST_LAUNCH("softmax_bwd_kernel");
  return MTKC_OK;
}

int mtkc_transpose(float* out, const float* src, const int64_t sd[4], const int perm[4],
                   int accumulate, void* stream) {
  TrP p;
  int64_t ss[4], run = 1;
  for(int i = 3; i >= 0; --i) {
    ss[i] = run;
    run *= sd[i];
  }
  p.n = run;
  for(int i = 0; i < 4; ++i) {
    p.od[i] = sd[perm[i]];
    p.ss[i] = ss[perm[i]];
  }
  p.out = out;
  p.src = src;
  p.acc = accumulate;
  if(p.n <= 0)
    return MTKC_OK;
  const bool vec = p.ss[3] == 1 && p.od[3] % 4 == 0 && p.ss[0] % 4 == 0 && p.ss[1] % 4 == 0 &&
                   p.ss[2] % 4 == 0 && (((uintptr_t)out | (uintptr_t)src) & 15) == 0;
  if(vec) {
    if(p.n / 4 < ((int64_t)1 << 31))
      ::mtkc::launch(transpose4_kernel<uint32_t>, grid1d(p.n / 4, 256), 256, 0, S(stream), p);
    else
      ::mtkc::launch(transpose4_kernel<int64_t>, grid1d(p.n / 4, 256), 256, 0, S(stream), p);
    MTKC_POST_LAUNCH("transpose4_kernel");
    return MTKC_OK;
  }
  ::mtkc::launch(transpose_kernel, grid1d(p.n, 256), 256, 0, S(stream), p);
  MTKC_POST_LAUNCH("transpose_kernel");
  return MTKC_OK;
}

int mtkc_copy_many(const mtkc_copy_job* jobs, int n, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  if(n > MTKC_COPY_MAX_JOBS)
    return fail(MTKC_CONTRACT, "mtkc_copy_many: too many jobs");
  CopyJobs cj{};
  int64_t most = 0;
  for(int i = 0; i < n; ++i) {
    cj.j[i] = jobs[i];
    most = std::max<int64_t>(most, jobs[i].rows * jobs[i].cols);
  }
  cj.n = n;
  ::mtkc::launch(copy_many_kernel, dim3(grid1d(most, 256, 148 * 4), (unsigned)n), 256, 0,
                 S(stream), cj);
  MTKC_POST_LAUNCH("copy_many_kernel");
  return MTKC_OK;
}

int mtkc_copy_blocks(float* dst, int64_t dst_stride, int64_t dst_off, const float* src,
                     int64_t src_stride, int64_t src_off, int64_t outer, int64_t len,
                     int accumulate, void* stream) {
  if(outer * len <= 0)
    return MTKC_OK;
  if(len % 4 == 0 && dst_stride % 4 == 0 && dst_off % 4 == 0 && src_stride % 4 == 0 &&
     src_off % 4 == 0 && (((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const int64_t n4 = outer * (len / 4);
    if(n4 < ((int64_t)1 << 31))
      ::mtkc::launch(copy_blocks4_kernel<uint32_t>, grid1d(n4, 256), 256, 0, S(stream), dst,
                     dst_stride, dst_off, src, src_stride, src_off, outer, len, accumulate);
    else
      ::mtkc::launch(copy_blocks4_kernel<int64_t>, grid1d(n4, 256), 256, 0, S(stream), dst,
                     dst_stride, dst_off, src, src_stride, src_off, outer, len, accumulate);
    MTKC_POST_LAUNCH("copy_blocks4_kernel");
    return MTKC_OK;
  }
  ::mtkc::launch(copy_blocks_kernel, grid1d(outer * len, 256), 256, 0, S(stream), 
      dst, dst_stride, dst_off, src, src_stride, src_off, outer, len, accumulate);
  MTKC_POST_LAUNCH("copy_blocks_kernel");
  return MTKC_OK;
}

int mtkc_gather_rows(float* out, const float* src, const int32_t* rows, int64_t n,
                     int64_t cols, int64_t src_rows, int* flags, void* stream) {
  if(n * cols <= 0)
    return MTKC_OK;
  ::mtkc::launch(gather_rows_kernel, grid1d(n * cols, 256), 256, 0, S(stream), out, src, rows, n, cols,
                                                                  src_rows, flags);
  MTKC_POST_LAUNCH("gather_rows_kernel");
  return MTKC_OK;
}

int mtkc_scatter_add_rows(float* out, const float* src, const int32_t* perm,
                          const int32_t* seg_start, const int32_t* uniq, int64_t n_uniq,
                          int64_t cols, float scale, void* stream) {
  if(n_uniq <= 0 || cols <= 0)
    return MTKC_OK;
  int threads = cols >= 256 ? 256 : (int)((cols + 31) / 32 * 32);
  ::mtkc::launch(scatter_add_kernel, (unsigned)n_uniq, threads, 0, S(stream), out, src, perm, seg_start,
                                                                  uniq, cols, scale);
  MTKC_POST_LAUNCH("scatter_add_kernel");
  return MTKC_OK;
}

int mtkc_scatter_add_rows_chunked(float* out, const float* src, const int32_t* perm,
                                  const int32_t* chunk_start, const int32_t* chunk_row,
                                  const int32_t* chunk_slot, int64_t n_chunks,
                                  const int32_t* multi_first, const int32_t* multi_row,
                                  int64_t n_multi, float* partial, int64_t cols, float scale,
                                  void* stream) {
  if(n_chunks <= 0 || cols <= 0)
    return MTKC_OK;
  int threads = cols >= 512 ? 512 : (int)((cols + 31) / 32 * 32);
  ::mtkc::launch(scatter_chunk_kernel, (unsigned)n_chunks, threads, 0, S(stream), 
      out, src, perm, chunk_start, chunk_row, chunk_slot, partial, cols, scale);
  MTKC_POST_LAUNCH("scatter_chunk_kernel");
  if(n_multi > 0) {
    ::mtkc::launch(scatter_multi_kernel, (unsigned)n_multi, threads, 0, S(stream), out, partial, multi_first,
                                                                       multi_row, cols);
    MTKC_POST_LAUNCH("scatter_multi_kernel");
  }
  return MTKC_OK;
}

int mtkc_embed(float* out, const float* table, const int32_t* ids, int64_t n, int64_t e,
               int64_t vocab, float s, const float* pe, int64_t t, int* flags, void* stream) {
  if(n * e <= 0)
    return MTKC_OK;
  if(t <= 0)
    t = 1;
  bool vec = e % 4 == 0 && (uintptr_t)out % 16 == 0 && (uintptr_t)table % 16 == 0 &&
             (!pe || (uintptr_t)pe % 16 == 0);
  if(vec)
    ::mtkc::launch(embed4_kernel, grid1d(n * e / 4, 256), 256, 0, S(stream), 
        (float4*)out, (const float4*)table, ids, n, e / 4, vocab, s, (const float4*)pe, t, flags,
        (const int32_t*)nullptr);
  else
    ::mtkc::launch(embed_kernel, grid1d(n * e, 256), 256, 0, S(stream), out, table, ids, n, e, vocab, s, pe,
                                                           t, flags);
  MTKC_POST_LAUNCH("embed_kernel");
  return MTKC_OK;
}

int mtkc_embed_pos(float* out, const float* table, const int32_t* ids, const int32_t* pos,
                   int64_t n, int64_t e, int64_t vocab, float s, const float* pe, int* flags,
                   void* stream) {
  if(n * e <= 0)
    return MTKC_OK;
  if(e % 4 || (uintptr_t)out % 16 || (uintptr_t)table % 16 || !pe || (uintptr_t)pe % 16)
    return fail(MTKC_DIMENSION, "mtkc_embed_pos: 16-byte aligned rows and a position table");
  ::mtkc::launch(embed4_kernel, grid1d(n * e / 4, 256), 256, 0, S(stream), (float4*)out,
                 (const float4*)table, ids, n, e / 4, vocab, s, (const float4*)pe, (int64_t)1,
                 flags, pos);
  MTKC_POST_LAUNCH("embed4_kernel");
  return MTKC_OK;
}

}  // extern "C"
