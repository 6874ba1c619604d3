// Reductions: reduceInto (tensor.cpp:322-368) and its graph backward
// (graph.cpp:488-521); deterministic column sums for bias/gain gradients;
// the allFinite scan (tensor.cpp:95-100) as a device flag.
#include "colred.cuh"
#include "common.cuh"

using namespace mtkc;

namespace {

__global__ void reduce_kernel(int op, float* out, const float* in, int64_t outer, int64_t n,
                              int64_t inner) {
  MTKC_PDL_ENTRY();
  int64_t total = outer * inner;
  for(int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
      t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = t / inner, c = t % inner;
    const float* base = in + a * n * inner + c;
    float acc;
    if(op == MTKC_RSUM || op == MTKC_RMEAN) {
      acc = 0.f;
      for(int64_t i = 0; i < n; ++i)
        acc += base[i * inner];
      if(op == MTKC_RMEAN)
        acc /= (float)n;
    } else if(op == MTKC_RMAX) {
      acc = base[0];
      for(int64_t i = 1; i < n; ++i)
        acc = fmaxf(acc, base[i * inner]);
    } else {
      float best = base[0];
      int64_t arg = 0;
      for(int64_t i = 1; i < n; ++i)
        if(base[i * inner] > best) {  // strict: ties keep the lowest index (:357)
          best = base[i * inner];
          arg = i;
        }
      acc = (float)arg;
    }
    out[t] = acc;
  }
}

__global__ void reduce_bwd_kernel(int op, float* gin, const float* gout, const float* in,
                                  int64_t outer, int64_t n, int64_t inner) {
  MTKC_PDL_ENTRY();
  int64_t total = outer * inner;
  for(int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
      t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = t / inner, c = t % inner;
    float go = gout[t];
    float* base = gin + a * n * inner + c;
    const float* xv = in + a * n * inner + c;
    if(op == MTKC_RSUM) {
      for(int64_t i = 0; i < n; ++i)
        base[i * inner] += go;
    } else if(op == MTKC_RMEAN) {
      float v = go / (float)n;
      for(int64_t i = 0; i < n; ++i)
        base[i * inner] += v;
    } else if(op == MTKC_RMAX) {
      int64_t best = 0;
      for(int64_t i = 1; i < n; ++i)
        if(xv[i * inner] > xv[best * inner])
          best = i;
      base[best * inner] += go;
    }
  }
}

constexpr int CS_ROWS = 128;  // below this many rows a single pass is used

// single-level variant (no workspace): one thread per column walks all rows
__global__ void colsum_direct_kernel(float* out, const float* in, int64_t rows, int64_t cols,
                                     int accumulate) {
  MTKC_PDL_ENTRY();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if(c >= cols)
    return;
  float s = 0.f;
  for(int64_t r = 0; r < rows; ++r)
    s += in[r * cols + c];
  out[c] = (accumulate ? out[c] : 0.f) + s;
}

// One-launch deterministic column sum: colred_partial_kernel's stage 1, then
// the last CTA to finish a 128-column slab (atomic ticket) sums that slab's
// row-block partials in fixed row-block order -- the result does not depend
// on which CTA is last.  Tickets reset themselves for the next call.
constexpr int CS_MAX_SLABS = 8192;
__device__ unsigned int g_colsum_ticket[CS_MAX_SLABS];

struct ColsumGroup {
  float* out[3];
  const float* in[3];
  int acc[3];
};

// gridDim.z = problems of a group (same shape): partial rows of problem z
// at part + z*nblk*cols, tickets at z*slabs + slab
__global__ void __launch_bounds__(256) colsum_onepass_kernel(ColsumGroup grp, float* part,
                                                             int64_t rows, int64_t cols) {
  MTKC_PDL_ENTRY();
  const int z = blockIdx.z;
  float* out = grp.out[z];
  const float* a = grp.in[z];
  const int acc = grp.acc[z];
  part += (int64_t)z * gridDim.y * cols;
  __shared__ float4 red[8][32];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * CR_COLS + lane * 4;
  const int64_t r0 = (int64_t)blockIdx.y * CR_ROWS + w;
  const int64_t nblk = gridDim.y;
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f);
  if(c < cols) {  // cols % 4 == 0 (host)
    float4 xa[CR_RPW];
#pragma unroll
    for(int i = 0; i < CR_RPW; ++i) {
      const int64_t r = r0 + 8 * i;
      xa[i] = r < rows ? __ldg(reinterpret_cast<const float4*>(a + r * cols + c))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for(int i = 0; i < CR_RPW; ++i)
      f4add(s0, xa[i]);
  }
  red[w][lane] = s0;
  __syncthreads();
  if(w == 0) {
    if(c < cols) {
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int k = 0; k < 8; ++k)
        f4add(t, red[k][lane]);
      *reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * cols + c) = t;
    }
    __threadfence();  // only the writers publish before the ticket
  }
  __syncthreads();
  if(threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&g_colsum_ticket[z * gridDim.x + blockIdx.x], 1u);
    last = prev == (unsigned)(nblk - 1);
  }
  __syncthreads();
  if(!last)
    return;
  __threadfence();
  // slab total: warp w sums row blocks w, w+8, ... (in order), then the 8
  // warps combine in fixed order
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if(c < cols)
    for(int64_t rb = w; rb < nblk; rb += 64) {  // eight loads in flight, summed in order
      float4 v[8];
#pragma unroll
      for(int u = 0; u < 8; ++u)
        v[u] = rb + 8 * u < nblk
                   ? __ldcg(reinterpret_cast<const float4*>(part + (rb + 8 * u) * cols + c))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int u = 0; u < 8; ++u)
        f4add(t, v[u]);
    }
  red[w][lane] = t;
  __syncthreads();
  if(w == 0) {
    if(c < cols) {
      float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int k = 0; k < 8; ++k)
        f4add(u, red[k][lane]);
      float4* o = reinterpret_cast<float4*>(out + c);
      if(acc) {
        float4 prevv = *o;
        u = make_float4(prevv.x + u.x, prevv.y + u.y, prevv.z + u.z, prevv.w + u.w);
      }
      *o = u;
    }
    if(lane == 0)
      g_colsum_ticket[z * gridDim.x + blockIdx.x] = 0u;
  }
}

// Several column sums over the same rows in one launch (the per-block bias
// and layer-norm gradient sums of the RNN scans): job z sums columns
// [0, cols) of a [rows x ld] matrix, stage 1 and the last-CTA slab finish
// exactly as colsum_onepass_kernel (same row blocks, same fixed order: the
// sums are bit-identical to one mtkc_colsum per job), and column c lands in
// segment c / seg: out[s][c % seg] (= or +=), or nowhere when out[s] is NULL.
struct ColsumMulti {
  mtkc_colsum_job j[MTKC_COLSUM_MAX_JOBS];
  int n;
  int slab0[MTKC_COLSUM_MAX_JOBS + 1];  // first global slab of each job
  int64_t part0[MTKC_COLSUM_MAX_JOBS];  // partial-row offset (floats) of each job
};

__global__ void __launch_bounds__(256) colsum_multi_kernel(const __grid_constant__ ColsumMulti m,
                                                           float* part, int64_t rows) {
  MTKC_PDL_ENTRY();
  int z = 0;
  while(z + 1 < m.n && (int)blockIdx.x >= m.slab0[z + 1])
    ++z;
  const mtkc_colsum_job& J = m.j[z];
  const int64_t cols = J.cols, ld = J.ld;
  part += m.part0[z];
  const int slab = (int)blockIdx.x - m.slab0[z];
  __shared__ float4 red[8][32];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)slab * CR_COLS + lane * 4;
  const int64_t r0 = (int64_t)blockIdx.y * CR_ROWS + w;
  const int64_t nblk = gridDim.y;
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f);
  if(c < cols) {
    float4 xa[CR_RPW];
#pragma unroll
    for(int i = 0; i < CR_RPW; ++i) {
      const int64_t r = r0 + 8 * i;
      xa[i] = r < rows ? __ldg(reinterpret_cast<const float4*>(J.in + r * ld + c))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for(int i = 0; i < CR_RPW; ++i)
      f4add(s0, xa[i]);
  }
  red[w][lane] = s0;
  __syncthreads();
  if(w == 0) {
    if(c < cols) {
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int k = 0; k < 8; ++k)
        f4add(t, red[k][lane]);
      *reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * cols + c) = t;
    }
    __threadfence();
  }
  __syncthreads();
  if(threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&g_colsum_ticket[blockIdx.x], 1u);
    last = prev == (unsigned)(nblk - 1);
  }
  __syncthreads();
  if(!last)
    return;
  __threadfence();
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if(c < cols)
    for(int64_t rb = w; rb < nblk; rb += 64) {
      float4 v[8];
#pragma unroll
      for(int u = 0; u < 8; ++u)
        v[u] = rb + 8 * u < nblk
                   ? __ldcg(reinterpret_cast<const float4*>(part + (rb + 8 * u) * cols + c))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int u = 0; u < 8; ++u)
        f4add(t, v[u]);
    }
  red[w][lane] = t;
  __syncthreads();
  if(w == 0) {
    if(c < cols) {
      float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for(int k = 0; k < 8; ++k)
        f4add(u, red[k][lane]);
      const int sg = (int)(c / J.seg);  // seg % 4 == 0: the 4 columns share a segment
      float* o = J.out[sg];
      if(o) {
        o += c - (int64_t)sg * J.seg;
        const float uu[4] = {u.x, u.y, u.z, u.w};
        for(int e = 0; e < 4; ++e)
          o[e] = J.acc[sg] ? o[e] + uu[e] : uu[e];
      }
    }
    if(lane == 0)
      g_colsum_ticket[blockIdx.x] = 0u;
  }
}

__global__ void colsum_multi_direct_kernel(const __grid_constant__ ColsumMulti m, int64_t rows) {
  MTKC_PDL_ENTRY();
  const mtkc_colsum_job& J = m.j[blockIdx.y];
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if(c >= J.cols)
    return;
  float s = 0.f;
  for(int64_t r = 0; r < rows; ++r)
    s += J.in[r * J.ld + c];
  const int sg = (int)(c / J.seg);
  float* o = J.out[sg];
  if(o) {
    o += c - (int64_t)sg * J.seg;
    *o = J.acc[sg] ? *o + s : s;
  }
}

__global__ void finite_kernel(const float* in, int64_t n, int* flags) {
  MTKC_PDL_ENTRY();
  bool bad = false;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
      i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(in[i]);
  if(__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(flags, MTKC_FLAG_NONFINITE);
}

__global__ void flag_or_kernel(int* dst, const int* src) {
  MTKC_PDL_ENTRY();
  if(threadIdx.x == 0 && *src)
    atomicOr(dst, *src);
}

__global__ void finite4_kernel(const float4* in, int64_t n4, int* flags) {
  MTKC_PDL_ENTRY();
  bool bad = false;
  for(int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
      i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = in[i];
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  if(__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(flags, MTKC_FLAG_NONFINITE);
}

}  // namespace

extern "C" {

int mtkc_reduce(int op, float* out, const float* in, int64_t outer, int64_t n, int64_t inner,
                void* stream) {
  if(outer * inner <= 0 || n <= 0)
    return MTKC_OK;
  ::mtkc::launch(reduce_kernel, grid1d(outer * inner, 128), 128, 0, S(stream), op, out, in, outer, n, inner);
  MTKC_POST_LAUNCH("reduce_kernel");
  return MTKC_OK;
}

int mtkc_reduce_backward(int op, float* gin, const float* gout, const float* in,
                         int64_t outer, int64_t n, int64_t inner, void* stream) {
  if(op == MTKC_RARGMAX || outer * inner <= 0)
    return MTKC_OK;
  ::mtkc::launch(reduce_bwd_kernel, grid1d(outer * inner, 128), 128, 0, S(stream), op, gin, gout, in, outer,
                                                                       n, inner);
  MTKC_POST_LAUNCH("reduce_bwd_kernel");
  return MTKC_OK;
}

int mtkc_colsum(float* out, const float* in, int64_t rows, int64_t cols, int accumulate,
                float* workspace, size_t workspace_bytes, void* stream) {
  if(rows <= 0 || cols <= 0)
    return MTKC_OK;
  ProfScope prof(S(stream), "colsum", 4.0 * rows * cols);
  if(prof_detail())
    prof.detail = "r" + std::to_string(rows) + "_c" + std::to_string(cols);
  const bool onepass = cols % 4 == 0 && rows > 8 && workspace &&
                       workspace_bytes >= colred_workspace_bytes(1, rows, cols);
  if(!onepass && (rows <= CS_ROWS || !workspace ||
                  workspace_bytes < colred_workspace_bytes(1, rows, cols))) {
    ::mtkc::launch(colsum_direct_kernel, (unsigned)cdiv(cols, 128), 128, 0, S(stream), out, in, rows, cols,
                                                                          accumulate);
    MTKC_POST_LAUNCH("colsum_direct_kernel");
    return MTKC_OK;
  }
  int64_t nblk = cdiv(rows, CR_ROWS);
  if(cols % 4 == 0 && cdiv(cols, CR_COLS) <= CS_MAX_SLABS && nblk <= 65535 &&
     ((uintptr_t)in | (uintptr_t)out | (uintptr_t)workspace) % 16 == 0) {
    ColsumGroup grp{};
    grp.out[0] = out;
    grp.in[0] = in;
    grp.acc[0] = accumulate;
    ::mtkc::launch(colsum_onepass_kernel, dim3((unsigned)cdiv(cols, CR_COLS), (unsigned)nblk), 256,
                   0, S(stream), grp, workspace, rows, cols);
    MTKC_POST_LAUNCH("colsum_onepass_kernel");
    return MTKC_OK;
  }
  ::mtkc::launch(colred_partial_kernel<1>, dim3((unsigned)cdiv(cols, CR_COLS), (unsigned)nblk), 256, 0,
                             S(stream), workspace, in, nullptr, rows, cols);
  MTKC_POST_LAUNCH("colred_partial_kernel");
  ::mtkc::launch(colred_final_kernel<1>, colred_final_grid(cols), 256, 0, S(stream), 
      out, nullptr, workspace, nblk, cols, accumulate);
  MTKC_POST_LAUNCH("colred_final_kernel");
  return MTKC_OK;
}

int mtkc_colsum_multi(const mtkc_colsum_job* jobs, int n, int64_t rows, float* workspace,
                      size_t workspace_bytes, void* stream) {
  if(n <= 0 || rows <= 0)
    return MTKC_OK;
  if(n > MTKC_COLSUM_MAX_JOBS)
    return fail(MTKC_CONTRACT, "mtkc_colsum_multi: too many jobs");
  ColsumMulti m{};
  m.n = n;
  const int64_t nblk = cdiv(rows, CR_ROWS);
  int64_t slabs = 0, partFloats = 0;
  double bytes = 0;
  bool ok = rows > 8 && nblk <= 65535 && workspace && (uintptr_t)workspace % 16 == 0;
  for(int z = 0; z < n && ok; ++z) {
    const mtkc_colsum_job& J = jobs[z];
    ok = J.cols > 0 && J.cols % 4 == 0 && J.ld % 4 == 0 && J.ld >= J.cols && J.seg > 0 &&
         J.seg % 4 == 0 && J.nseg >= (int)cdiv(J.cols, J.seg) && J.nseg <= MTKC_COLSUM_MAX_SEGS &&
         (uintptr_t)J.in % 16 == 0;
    m.j[z] = J;
    m.slab0[z] = (int)slabs;
    m.part0[z] = partFloats;
    slabs += cdiv(J.cols, CR_COLS);
    partFloats += nblk * J.cols;
    bytes += 4.0 * rows * J.cols;
  }
  m.slab0[n] = (int)slabs;
  ok = ok && slabs <= CS_MAX_SLABS && (size_t)partFloats * sizeof(float) <= workspace_bytes;
  ProfScope prof(S(stream), "colsum", bytes);
  if(!ok) {  // few rows / odd shapes: one thread per column, rows in order
    int64_t maxc = 0;
    for(int z = 0; z < n; ++z) {
      m.j[z] = jobs[z];
      if(jobs[z].seg <= 0 || jobs[z].nseg * jobs[z].seg < jobs[z].cols)
        return fail(MTKC_CONTRACT, "mtkc_colsum_multi: segments do not cover the columns");
      maxc = std::max(maxc, jobs[z].cols);
    }
    ::mtkc::launch(colsum_multi_direct_kernel, dim3((unsigned)cdiv(maxc, 128), (unsigned)n), 128,
                   0, S(stream), m, rows);
    MTKC_POST_LAUNCH("colsum_multi_direct_kernel");
    return MTKC_OK;
  }
  if(prof_detail())
    prof.detail = "multi" + std::to_string(n) + "_r" + std::to_string(rows);
  ::mtkc::launch(colsum_multi_kernel, dim3((unsigned)slabs, (unsigned)nblk), 256, 0, S(stream), m,
                 workspace, rows);
  MTKC_POST_LAUNCH("colsum_multi_kernel");
  return MTKC_OK;
}

int mtkc_colsum_group(float* const* outs, const float* const* ins, const int* accumulate, int n,
                      int64_t rows, int64_t cols, float* workspace, size_t workspace_bytes,
                      void* stream) {
  if(n < 1 || rows <= 0 || cols <= 0)
    return MTKC_OK;
  const int64_t nblk = cdiv(rows, CR_ROWS), slabs = cdiv(cols, CR_COLS);
  bool ok = n <= 3 && cols % 4 == 0 && rows > 8 && slabs * n <= CS_MAX_SLABS && nblk <= 65535 &&
            workspace && workspace_bytes >= (size_t)n * colred_workspace_bytes(1, rows, cols) &&
            (uintptr_t)workspace % 16 == 0;
  for(int q = 0; q < n && ok; ++q)
    ok = ((uintptr_t)ins[q] | (uintptr_t)outs[q]) % 16 == 0;
  if(!ok) {  // one problem at a time
    for(int q = 0; q < n; ++q)
      if(int rc = mtkc_colsum(outs[q], ins[q], rows, cols, accumulate[q], workspace,
                              workspace_bytes, stream))
        return rc;
    return MTKC_OK;
  }
  ProfScope prof(S(stream), "colsum", 4.0 * n * rows * cols);
  if(prof_detail())
    prof.detail = "group" + std::to_string(n) + "_r" + std::to_string(rows) + "_c" +
                  std::to_string(cols);
  ColsumGroup grp{};
  for(int q = 0; q < n; ++q) {
    grp.out[q] = outs[q];
    grp.in[q] = ins[q];
    grp.acc[q] = accumulate[q];
  }
  ::mtkc::launch(colsum_onepass_kernel, dim3((unsigned)slabs, (unsigned)nblk, (unsigned)n), 256, 0,
                 S(stream), grp, workspace, rows, cols);
  MTKC_POST_LAUNCH("colsum_onepass_kernel");
  return MTKC_OK;
}

int mtkc_flag_or(int* dst, const int* src, void* stream) {
  ::mtkc::launch(flag_or_kernel, 1, 32, 0, S(stream), dst, src);
  MTKC_POST_LAUNCH("flag_or_kernel");
  return MTKC_OK;
}

int mtkc_check_finite(const float* in, int64_t n, int* flags, void* stream) {
  if(n <= 0)
    return MTKC_OK;
  if(n % 4 == 0 && (uintptr_t)in % 16 == 0)
    ::mtkc::launch(finite4_kernel, grid1d(n / 4, 256, 148 * 8), 256, 0, S(stream), (const float4*)in, n / 4,
                                                                      flags);
  else
    ::mtkc::launch(finite_kernel, grid1d(n, 256, 148 * 8), 256, 0, S(stream), in, n, flags);
  MTKC_POST_LAUNCH("finite_kernel");
  return MTKC_OK;
}

}  // extern "C"
