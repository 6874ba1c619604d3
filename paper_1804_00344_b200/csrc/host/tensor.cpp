// Device tensors, the device arena and the tensor-level kernel wrappers
// (reference: src/tensor.cpp).  Shape checks and their messages follow the
// reference; the arithmetic runs in libmtkcuda.so.
#include "mtk/tensor.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>

#include "mtk/device.h"

namespace mtk {

// ---------------------------------------------------------------- Shape

void Shape::validate() const {
  if(dims_.empty() || dims_.size() > 4)
    throw DimensionError("shape rank must be 1..4, got rank " + std::to_string(dims_.size()));
  for(auto d : dims_)
    if(d < 1)
      throw DimensionError("shape extents must be >= 1, got " + str());
}

std::string Shape::str() const {
  std::ostringstream os;
  os << "[";
  for(size_t i = 0; i < dims_.size(); ++i)
    os << (i ? "x" : "") << dims_[i];
  os << "]";
  return os.str();
}

void Shape::pad4(int64_t out[4]) const {
  out[0] = out[1] = out[2] = out[3] = 1;
  int off = 4 - rank();
  for(int i = 0; i < rank(); ++i)
    out[off + i] = dims_[(size_t)i];
}

// --------------------------------------------------------- DeviceBuffer

// Caching device allocator: cudaMalloc/cudaFree synchronise the device, so
// steady-state training must never call them.  Freed blocks go to a size-
// keyed free list and are reused.  Small blocks (batch masks, index vectors:
// a new batch shape brings new sizes) are carved from 64 MB slabs in
// power-of-two / 1.5x size classes, so a size first seen inside a timed
// step costs no cudaMalloc.  Every kernel runs on the one compute stream, so
// a block released by the host may be handed out again at once: work queued
// later on the stream runs after all work that used it.
namespace {
struct BlockCache {
  static constexpr size_t SMALL = (size_t)1 << 20, SLAB = (size_t)64 << 20;
  std::map<size_t, std::vector<void*>> free;
  char* slab = nullptr;
  size_t slabLeft = 0;
  static size_t round(size_t bytes) {
    if(bytes <= SMALL) {
      size_t p = 512;
      while(p < bytes) {
        if(p >= 1024 && p + p / 2 >= bytes)
          return p + p / 2;
        p <<= 1;
      }
      return p;
    }
    return (bytes + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
  }
  void* take(size_t bytes) {
    if(bytes > SMALL) {
      void* p = nullptr;
      MTKC(mtkc_malloc(&p, bytes));
      return p;
    }
    if(slabLeft < bytes) {
      void* p = nullptr;
      MTKC(mtkc_malloc(&p, SLAB));
      slab = (char*)p;
      slabLeft = SLAB;
    }
    void* p = slab;
    slab += bytes;
    slabLeft -= bytes;
    return p;
  }
};
BlockCache& cache() {
  static BlockCache* c = new BlockCache();  // process lifetime
  return *c;
}
}  // namespace

DeviceBuffer::DeviceBuffer(size_t n) : elems(n) {
  Device::get();
  size_t bytes = BlockCache::round(std::max<size_t>(n, 1) * sizeof(float));
  auto& fl = cache().free[bytes];
  if(!fl.empty()) {
    ptr = (float*)fl.back();
    fl.pop_back();
    return;
  }
  ptr = (float*)cache().take(bytes);
}

DeviceBuffer::~DeviceBuffer() {
  if(owned && ptr)
    cache().free[BlockCache::round(std::max<size_t>(elems, 1) * sizeof(float))].push_back(ptr);
}

// ---------------------------------------------------------------- Tensor

Tensor::Tensor(Shape shape) : shape_(std::move(shape)) {
  host_ = std::make_shared<HostCache>();
  host_->data.assign((size_t)shape_.size(), Real(0));
  host_->valid = true;
  host_->dirty = true;
}

Tensor::Tensor(Shape shape, std::vector<Real> values) : shape_(std::move(shape)) {
  if((int64_t)values.size() != shape_.size())
    throw DimensionError("tensor data length " + std::to_string(values.size()) +
                         " does not match shape " + shape_.str());
  host_ = std::make_shared<HostCache>();
  host_->data = std::move(values);
  host_->valid = true;
  host_->dirty = true;
}

Tensor::Tensor(Shape shape, std::shared_ptr<DeviceBuffer> buf, int64_t offset)
    : shape_(std::move(shape)), buf_(std::move(buf)), off_(offset) {
  if(!buf_)
    throw ContractError("tensor view over null storage");
}

void Tensor::ensureDevice() const {
  if(!buf_) {
    if(host_ && host_->devbuf) {  // another copy of this tensor already uploaded
      buf_ = host_->devbuf;
      off_ = 0;
    } else {
      buf_ = std::make_shared<DeviceBuffer>((size_t)size());
      off_ = 0;
      if(host_)
        host_->devbuf = buf_;
      if(!host_ || !host_->valid)
        MTKC(mtkc_memset(buf_->ptr, 0, (size_t)size() * sizeof(float), Device::get().stream()));
    }
  }
  if(host_ && host_->dirty) {
    Device::get().upload(buf_->ptr + off_, host_->data.data(), (size_t)size() * sizeof(float));
    host_->dirty = false;
  }
}

float* Tensor::dev() const {
  if(empty())
    throw ContractError("device access to an empty tensor");
  ensureDevice();
  if(host_)
    host_->valid = false;
  return buf_->ptr + off_;
}

const float* Tensor::devc() const {
  if(empty())
    throw ContractError("device access to an empty tensor");
  ensureDevice();
  return buf_->ptr + off_;
}

void Tensor::ensureHost() const {
  if(!host_)
    host_ = std::make_shared<HostCache>();
  if(host_->valid)
    return;
  host_->data.resize((size_t)size());
  if(buf_) {
    Device& d = Device::get();
    MTKC(mtkc_memcpy_d2h(host_->data.data(), buf_->ptr + off_, (size_t)size() * sizeof(float),
                         d.stream()));
    d.checkFlags("tensor read");
  }
  host_->valid = true;
}

Real* Tensor::data() {
  if(empty())
    return nullptr;
  ensureHost();
  host_->dirty = true;
  return host_->data.data();
}

const Real* Tensor::data() const {
  if(empty())
    return nullptr;
  ensureHost();
  return host_->data.data();
}

Tensor Tensor::copy() const {
  if(!buf_) {
    Tensor out(shape_, host_ ? host_->data : std::vector<Real>((size_t)size(), 0));
    return out;
  }
  auto nb = std::make_shared<DeviceBuffer>((size_t)size());
  MTKC(mtkc_memcpy_d2d(nb->ptr, devc(), (size_t)size() * sizeof(float), Device::get().stream()));
  return Tensor(shape_, nb, 0);
}

void Tensor::setZero() {
  if(empty())
    return;
  if(!buf_) {
    std::fill(host_->data.begin(), host_->data.end(), Real(0));
    host_->valid = true;
    host_->dirty = true;
    return;
  }
  if(host_)
    host_->dirty = false;
  MTKC(mtkc_memset(dev(), 0, (size_t)size() * sizeof(float), Device::get().stream()));
}

void Tensor::fill(Real v) {
  if(empty())
    return;
  if(!buf_) {
    std::fill(host_->data.begin(), host_->data.end(), v);
    host_->valid = true;
    host_->dirty = true;
    return;
  }
  if(host_)
    host_->dirty = false;
  MTKC(mtkc_fill(dev(), v, size(), Device::get().stream()));
}

void Tensor::copyFrom(const Tensor& src) {
  if(src.size() != size())
    throw DimensionError("copyFrom size mismatch " + src.shape().str() + " vs " + shape_.str());
  if(!buf_ && !src.buf_) {
    host_->data = src.toVector();
    host_->valid = true;
    host_->dirty = true;
    return;
  }
  if(host_)
    host_->dirty = false;
  MTKC(mtkc_memcpy_d2d(dev(), src.devc(), (size_t)size() * sizeof(float), Device::get().stream()));
}

std::vector<Real> Tensor::toVector() const {
  const Real* p = data();
  return std::vector<Real>(p, p + size());
}

bool Tensor::allFinite() const {
  const Real* p = data();
  for(int64_t i = 0; i < size(); ++i)
    if(!std::isfinite(p[i]))
      return false;
  return true;
}

Tensor Tensor::reshaped(Shape s) const {
  if(s.size() != size())
    throw DimensionError("reshape element count mismatch: " + shape_.str() + " -> " + s.str());
  ensureDevice();
  Tensor t(std::move(s), buf_, off_);
  t.host_ = host_;  // same storage, same cache
  return t;
}

// ----------------------------------------------------------------- Arena

std::pair<std::shared_ptr<DeviceBuffer>, int64_t> Arena::alloc(int64_t elements) {
  if(elements <= 0)
    throw ContractError("arena alloc of non-positive size");
  size_t n = ((size_t)elements + 63) & ~(size_t)63;  // 256-byte granularity
  size_t bytes = n * sizeof(float);
  if(outstanding_ + bytes > capacity_)
    throw NumericError("arena capacity exceeded: " + std::to_string(outstanding_ + bytes) +
                       " > " + std::to_string(capacity_) + " bytes");
  while(cur_ < slabs_.size() && slabs_[cur_].used + n > slabs_[cur_].buf->elems)
    ++cur_;
  if(cur_ == slabs_.size()) {
    // geometric growth (each new slab as large as everything reserved so
    // far, 256 MiB .. 4 GiB): a few cudaMallocs instead of one per 256 MiB
    size_t grow = std::min<size_t>(std::max<size_t>(reservedBytes(), (size_t)256 << 20),
                                   (size_t)4 << 30);
    size_t slabElems = std::max(n, grow / sizeof(float));
    slabs_.push_back(Slab{std::make_shared<DeviceBuffer>(slabElems), 0});
  }
  Slab& s = slabs_[cur_];
  int64_t off = (int64_t)s.used;
  s.used += n;
  outstanding_ += bytes;
  highWater_ = std::max(highWater_, outstanding_);
  return {s.buf, off};
}

void Arena::reset() {
  for(auto& s : slabs_)
    s.used = 0;
  cur_ = 0;
  outstanding_ = 0;
}

size_t Arena::reservedBytes() const {
  size_t b = 0;
  for(auto& s : slabs_)
    b += s.buf->elems * sizeof(float);
  return b;
}

// ------------------------------------------------------------ broadcast

Shape broadcastShape(const Shape& a, const Shape& b) {
  int64_t da[4], db[4];
  a.pad4(da);
  b.pad4(db);
  std::vector<int64_t> out;
  for(int i = 0; i < 4; ++i) {
    if(da[i] == db[i] || da[i] == 1 || db[i] == 1)
      out.push_back(std::max(da[i], db[i]));
    else
      throw DimensionError("shapes not broadcastable: " + a.str() + " vs " + b.str());
  }
  int rank = std::max(a.rank(), b.rank());
  return Shape(std::vector<int64_t>(out.end() - rank, out.end()));
}

static void checkBroadcastInto(const Shape& operand, const Shape& out) {
  int64_t d[4], o[4];
  operand.pad4(d);
  out.pad4(o);
  for(int i = 0; i < 4; ++i)
    if(d[i] != 1 && d[i] != o[i])
      throw DimensionError("operand shape " + operand.str() + " incompatible with broadcast result");
}

static int opId(EwiseOp op) { return (int)op; }

void ewiseBinaryInto(Tensor& out, EwiseOp op, const Tensor& a, const Tensor& b) {
  checkBroadcastInto(a.shape(), out.shape());
  checkBroadcastInto(b.shape(), out.shape());
  int64_t od[4], ad[4], bd[4];
  out.shape().pad4(od);
  a.shape().pad4(ad);
  b.shape().pad4(bd);
  Device& d = Device::get();
  MTKC(mtkc_ewise_binary(opId(op), out.dev(), od, a.devc(), ad, b.devc(), bd, d.flags(),
                         d.stream()));
}

void ewiseUnaryInto(Tensor& out, EwiseOp op, const Tensor& a) {
  MTKC(mtkc_ewise_unary(opId(op), out.dev(), a.devc(), a.size(), Device::get().stream()));
}

Tensor ewise(EwiseOp op, const Tensor& a, const Tensor& b) {
  if(op == EwiseOp::Div) {  // tensor.cpp:161-165: checked eagerly on the host copy
    for(Real v : b.toVector())
      if(v == Real(0))
        throw NumericError("division by zero in elementwise div");
  }
  Tensor out(broadcastShape(a.shape(), b.shape()));
  ewiseBinaryInto(out, op, a, b);
  return out;
}

Tensor ewise(EwiseOp op, const Tensor& a) {
  Tensor out(a.shape());
  ewiseUnaryInto(out, op, a);
  return out;
}

void accumulateReduced(Tensor& out, const Tensor& src) {
  int64_t od[4], sd[4];
  out.shape().pad4(od);
  src.shape().pad4(sd);
  if(out.shape() == src.shape()) {
    axpy(out, src);
    return;
  }
  checkBroadcastInto(out.shape(), src.shape());
  MTKC(mtkc_accumulate_reduced(out.dev(), od, src.devc(), sd, Device::get().stream()));
}

void axpy(Tensor& out, const Tensor& a, Real alpha) {
  if(out.size() != a.size())
    throw DimensionError("axpy size mismatch");
  MTKC(mtkc_axpy(out.dev(), a.devc(), alpha, a.size(), Device::get().stream()));
}

// -------------------------------------------------------------- matmul

namespace {
struct MatView {
  int64_t batch, rows, cols, batchStride, ld;
};

MatView matView(const Tensor& t, bool trans) {
  const Shape& s = t.shape();
  if(s.rank() == 2)
    return {1, trans ? s[1] : s[0], trans ? s[0] : s[1], 0, s[1]};
  if(s.rank() == 3)
    return {s[0], trans ? s[2] : s[1], trans ? s[1] : s[2], s[1] * s[2], s[2]};
  throw DimensionError("matmul operands must be rank 2 or 3, got " + s.str());
}
}  // namespace

void matmulInto(Tensor& c, const Tensor& a, const Tensor& b, bool transA, bool transB,
                Real alpha, Real beta) {
  MatView va = matView(a, transA), vb = matView(b, transB);
  if(va.cols != vb.rows)
    throw DimensionError("matmul inner dims disagree: " + a.shape().str() + " x " +
                         b.shape().str());
  int64_t batch = std::max(va.batch, vb.batch);
  if(va.batch != vb.batch && va.batch != 1 && vb.batch != 1)
    throw DimensionError("matmul batch dims disagree: " + a.shape().str() + " x " +
                         b.shape().str());
  int64_t m = va.rows, k = va.cols, n = vb.cols;
  if(c.size() != batch * m * n)
    throw DimensionError("matmul output size mismatch");
  Device& d = Device::get();
  mtkc_gemm_args g{};
  g.M = m;
  g.N = n;
  g.K = k;
  g.batch = batch;
  g.A = a.devc();
  g.lda = va.ld;
  g.strideA = va.batch == 1 ? 0 : va.batchStride;
  g.transA = transA;
  g.B = b.devc();
  g.ldb = vb.ld;
  g.strideB = vb.batch == 1 ? 0 : vb.batchStride;
  g.transB = transB;
  g.C = c.dev();
  g.ldc = n;
  g.strideC = m * n;
  g.alpha = alpha;
  g.beta = beta;
  g.precision = (int)d.precision();
  g.workspace = d.scratch(64 << 20);
  g.workspace_bytes = d.scratchBytes();
  MTKC(mtkc_gemm(&g, d.stream()));
}

Tensor matmul(const Tensor& a, const Tensor& b, bool transA, bool transB) {
  MatView va = matView(a, transA), vb = matView(b, transB);
  int64_t batch = std::max(va.batch, vb.batch);
  Shape out = (a.shape().rank() == 3 || b.shape().rank() == 3)
                  ? Shape({batch, va.rows, vb.cols})
                  : Shape({va.rows, vb.cols});
  Tensor c(out);
  matmulInto(c, a, b, transA, transB);
  return c;
}

// ------------------------------------------------------------- reduce

void reduceInto(Tensor& out, ReduceOp op, const Tensor& t, int axis, bool keepAxis) {
  (void)keepAxis;
  int rank = t.shape().rank();
  if(axis < 0 || axis >= rank)
    throw DimensionError("reduce axis " + std::to_string(axis) + " out of range for " +
                         t.shape().str());
  int64_t outer = 1, inner = 1, n = t.shape()[axis];
  for(int i = 0; i < axis; ++i)
    outer *= t.shape()[i];
  for(int i = axis + 1; i < rank; ++i)
    inner *= t.shape()[i];
  MTKC(mtkc_reduce((int)op, out.dev(), t.devc(), outer, n, inner, Device::get().stream()));
}

Tensor reduce(ReduceOp op, const Tensor& t, int axis, bool keepAxis) {
  int rank = t.shape().rank();
  if(axis < 0 || axis >= rank)
    throw DimensionError("reduce axis " + std::to_string(axis) + " out of range for " +
                         t.shape().str());
  std::vector<int64_t> dims;
  for(int i = 0; i < rank; ++i) {
    if(i == axis) {
      if(keepAxis)
        dims.push_back(1);
    } else {
      dims.push_back(t.shape()[i]);
    }
  }
  if(dims.empty())
    dims.push_back(1);
  Tensor out((Shape(dims)));
  reduceInto(out, op, t, axis, keepAxis);
  return out;
}

// ------------------------------------------------------------- softmax

void softmaxInto(Tensor& out, const Tensor& t, const Tensor* mask, bool logMode) {
  int64_t xd[4], md[4] = {1, 1, 1, 1};
  t.shape().pad4(xd);
  const float* mp = nullptr;
  if(mask && !mask->empty()) {
    checkBroadcastInto(mask->shape(), t.shape());
    mask->shape().pad4(md);
    mp = mask->devc();
  }
  Device& d = Device::get();
  MTKC(mtkc_softmax(out.dev(), t.devc(), xd, mp, md, logMode ? 1 : 0, d.flags(), d.stream()));
}

Tensor softmax(const Tensor& t, const Tensor* mask) {
  Tensor out(t.shape());
  softmaxInto(out, t, mask, false);
  Device::get().checkFlags("softmax");
  return out;
}

Tensor logSoftmax(const Tensor& t, const Tensor* mask) {
  Tensor out(t.shape());
  softmaxInto(out, t, mask, true);
  Device::get().checkFlags("logSoftmax");
  return out;
}

// -------------------------------------------------- gather / scatter

namespace {
// Upload int ids to a transient device buffer (stream-ordered; the host
// vector stays alive until the copy is issued from pageable memory).
std::shared_ptr<DeviceBuffer> uploadInts(const std::vector<int32_t>& v) {
  auto b = std::make_shared<DeviceBuffer>(std::max<size_t>(v.size(), 1));
  MTKC(mtkc_memcpy_h2d(b->ptr, v.data(), v.size() * sizeof(int32_t), Device::get().stream()));
  return b;
}
}  // namespace

void gatherRowsInto(Tensor& out, const Tensor& src, const std::vector<int64_t>& rows) {
  int64_t cols = src.size() / src.shape()[0];
  int64_t nrows = src.shape()[0];
  std::vector<int32_t> r32(rows.size());
  for(size_t i = 0; i < rows.size(); ++i) {
    if(rows[i] < 0 || rows[i] >= nrows)
      throw ContractError("row index " + std::to_string(rows[i]) + " out of range 0.." +
                          std::to_string(nrows - 1));
    r32[i] = (int32_t)rows[i];
  }
  auto ids = uploadInts(r32);
  Device& d = Device::get();
  MTKC(mtkc_gather_rows(out.dev(), src.devc(), (const int32_t*)ids->ptr, (int64_t)rows.size(),
                        cols, nrows, d.flags(), d.stream()));
  d.sync();  // ids buffer released below
}

void scatterAddRows(Tensor& out, const Tensor& src, const std::vector<int64_t>& rows) {
  int64_t cols = out.size() / out.shape()[0];
  // stable sort of positions by row id -> segments summed in position order
  std::vector<int32_t> perm(rows.size());
  for(size_t i = 0; i < rows.size(); ++i)
    perm[i] = (int32_t)i;
  std::stable_sort(perm.begin(), perm.end(),
                   [&](int32_t x, int32_t y) { return rows[(size_t)x] < rows[(size_t)y]; });
  std::vector<int32_t> seg, uniq;
  for(size_t k = 0; k < perm.size(); ++k)
    if(k == 0 || rows[(size_t)perm[k]] != rows[(size_t)perm[k - 1]]) {
      seg.push_back((int32_t)k);
      uniq.push_back((int32_t)rows[(size_t)perm[k]]);
    }
  seg.push_back((int32_t)perm.size());
  auto p = uploadInts(perm), s = uploadInts(seg), u = uploadInts(uniq);
  Device& d = Device::get();
  MTKC(mtkc_scatter_add_rows(out.dev(), src.devc(), (const int32_t*)p->ptr,
                             (const int32_t*)s->ptr, (const int32_t*)u->ptr,
                             (int64_t)uniq.size(), cols, 1.f, d.stream()));
  d.sync();
}

// -------------------------------------------- transpose / concat / slice

void transposeInto(Tensor& out, const Tensor& src, const std::vector<int>& perm) {
  int rank = src.shape().rank();
  if((int)perm.size() != rank)
    throw DimensionError("transpose perm rank mismatch");
  int64_t sd[4];
  src.shape().pad4(sd);
  int off = 4 - rank;
  int p4[4] = {0, 1, 2, 3};
  for(int i = 0; i < rank; ++i)
    p4[off + i] = off + perm[(size_t)i];
  MTKC(mtkc_transpose(out.dev(), src.devc(), sd, p4, 0, Device::get().stream()));
}

void concatInto(Tensor& out, const std::vector<const Tensor*>& parts, int axis) {
  int rank = out.shape().rank();
  int64_t outer = 1, inner = 1;
  for(int i = 0; i < axis; ++i)
    outer *= out.shape()[i];
  for(int i = axis + 1; i < rank; ++i)
    inner *= out.shape()[i];
  int64_t outAxis = out.shape()[axis];
  int64_t offset = 0;
  float* o = out.dev();
  for(const Tensor* p : parts) {
    int64_t pa = p->shape()[axis];
    MTKC(mtkc_copy_blocks(o, outAxis * inner, offset * inner, p->devc(), pa * inner, 0, outer,
                          pa * inner, 0, Device::get().stream()));
    offset += pa;
  }
}

void sliceInto(Tensor& out, const Tensor& src, int axis, int64_t start, int64_t len) {
  int rank = src.shape().rank();
  int64_t outer = 1, inner = 1;
  for(int i = 0; i < axis; ++i)
    outer *= src.shape()[i];
  for(int i = axis + 1; i < rank; ++i)
    inner *= src.shape()[i];
  int64_t n = src.shape()[axis];
  if(start < 0 || start + len > n)
    throw DimensionError("slice out of range");
  MTKC(mtkc_copy_blocks(out.dev(), len * inner, 0, src.devc(), n * inner, start * inner, outer,
                        len * inner, 0, Device::get().stream()));
}

// ----------------------------------------------------------- layer norm

void layerNormInto(Tensor& out, const Tensor& x, const Tensor& gain, const Tensor& bias,
                   Real eps, Tensor& invStd, Tensor& xhat) {
  int64_t d = x.shape().back();
  int64_t rows = x.size() / d;
  MTKC(mtkc_layernorm(out.dev(), x.devc(), gain.devc(), bias.devc(), eps, invStd.dev(),
                      xhat.dev(), rows, d, Device::get().stream()));
}

void layerNormBackward(const Tensor& dy, const Tensor& gain, const Tensor& invStd,
                       const Tensor& xhat, Tensor& dx, Tensor& dgain, Tensor& dbias) {
  int64_t d = dy.shape().back();
  int64_t rows = dy.size() / d;
  Device& dev = Device::get();
  size_t ws = (size_t)((rows + 63) / 64) * 2 * (size_t)d * sizeof(float);
  float* w = dev.scratch(ws);
  MTKC(mtkc_layernorm_backward(dy.devc(), gain.devc(), invStd.devc(), xhat.devc(), dx.dev(),
                               dgain.dev(), dbias.dev(), rows, d, 1, 1, w, dev.scratchBytes(),
                               dev.stream()));
}

}  // namespace mtk
