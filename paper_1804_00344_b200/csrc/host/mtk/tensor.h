// Device-resident tensors and the device workspace arena.
//
// Reference: include/mtk/tensor.h (Shape :14-38, Arena :43-61, Tensor
// :65-98).  The public surface is kept -- Shape is identical, Tensor keeps
// data()/at()/copy()/setZero()/fill()/copyFrom()/toVector()/allFinite() --
// but storage is HBM:
//   * a Tensor is a view (device buffer + element offset) with a host cache
//     shared by all copies of that view.  Host accessors synchronise the
//     compute stream and download; host writes mark the cache dirty and are
//     uploaded before the next device use.  Tensors built from host data
//     (masks, constants) live on the host until first device use.
//   * the Arena hands out 256-byte aligned slices of device memory from a
//     list of slabs that survive reset(), so replaying one step's
//     allocation sequence reuses the same addresses and the high-water mark
//     stabilises after the first step (tensor.cpp:30-59 semantics; capacity
//     overflow is a NumericError).
#pragma once

#include <map>
#include <memory>
#include <vector>

#include "mtk/common.h"

namespace mtk {

class Shape {
public:
  Shape() = default;
  Shape(std::initializer_list<int64_t> dims) : dims_(dims) { validate(); }
  explicit Shape(std::vector<int64_t> dims) : dims_(std::move(dims)) { validate(); }

  int rank() const { return (int)dims_.size(); }
  int64_t operator[](int i) const { return dims_[(size_t)i]; }
  int64_t size() const {
    int64_t n = 1;
    for(auto d : dims_)
      n *= d;
    return n;
  }
  const std::vector<int64_t>& dims() const { return dims_; }
  int64_t back() const { return dims_.back(); }
  bool operator==(const Shape& o) const { return dims_ == o.dims_; }
  bool operator!=(const Shape& o) const { return dims_ != o.dims_; }
  std::string str() const;
  // right-aligned rank-4 padding (tensor.cpp:102-108)
  void pad4(int64_t out[4]) const;

private:
  void validate() const;
  std::vector<int64_t> dims_;
};

// Owned device allocation.  `ptr` may be swapped in place when a pool grows
// so every view follows (see ParamPool).
struct DeviceBuffer {
  float* ptr = nullptr;
  size_t elems = 0;
  bool owned = true;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n);
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

class Tensor {
public:
  Tensor() = default;
  explicit Tensor(Shape shape);                  // zeros (host-staged)
  Tensor(Shape shape, std::vector<Real> values);  // host-staged
  // view of device memory (buf->ptr + offset)
  Tensor(Shape shape, std::shared_ptr<DeviceBuffer> buf, int64_t offset);

  bool empty() const { return !buf_ && !host_; }
  const Shape& shape() const { return shape_; }
  int64_t size() const { return shape_.size(); }

  // --- host accessors (synchronise the stream on first read after a device write)
  Real* data();
  const Real* data() const;
  Real& at(int64_t i) { return data()[i]; }
  Real at(int64_t i) const { return data()[i]; }
  Tensor copy() const;  // deep copy into a new device buffer
  void setZero();
  void fill(Real v);
  void copyFrom(const Tensor& src);  // same element count required
  std::vector<Real> toVector() const;
  bool allFinite() const;

  // --- device accessors
  float* dev() const;         // may be written by the caller: invalidates the host cache
  const float* devc() const;  // read-only device access
  bool onDevice() const { return (bool)buf_; }
  // a reshaped view of the same storage (no copy)
  Tensor reshaped(Shape s) const;

private:
  struct HostCache {
    std::vector<Real> data;
    bool valid = false;
    bool dirty = false;
    std::shared_ptr<DeviceBuffer> devbuf;  // device copy shared by all copies of the tensor
  };
  void ensureDevice() const;
  void ensureHost() const;
  Shape shape_;
  mutable std::shared_ptr<DeviceBuffer> buf_;
  mutable int64_t off_ = 0;
  mutable std::shared_ptr<HostCache> host_;
};

// Device workspace allocator for one graph.
class Arena {
public:
  explicit Arena(size_t capacityBytes = (size_t)1 << 33) : capacity_(capacityBytes) {}
  // returns a view-able slice: (buffer, element offset)
  std::pair<std::shared_ptr<DeviceBuffer>, int64_t> alloc(int64_t elements);
  void reset();
  size_t capacity() const { return capacity_; }
  size_t outstandingBytes() const { return outstanding_; }
  size_t highWaterBytes() const { return highWater_; }
  size_t reservedBytes() const;

private:
  struct Slab {
    std::shared_ptr<DeviceBuffer> buf;
    size_t used = 0;  // elements
  };
  size_t capacity_;
  size_t outstanding_ = 0;
  size_t highWater_ = 0;
  std::vector<Slab> slabs_;
  size_t cur_ = 0;
};

enum class EwiseOp { Add, Sub, Mul, Div, Tanh, Sigmoid, Relu, Exp, Log, Neg };
enum class ReduceOp { Sum, Max, Mean, Argmax };

Shape broadcastShape(const Shape& a, const Shape& b);

// --- allocating front-end ops (tensor.h:108-114), executed on the device
Tensor matmul(const Tensor& a, const Tensor& b, bool transA = false, bool transB = false);
Tensor ewise(EwiseOp op, const Tensor& a, const Tensor& b);
Tensor ewise(EwiseOp op, const Tensor& a);
Tensor reduce(ReduceOp op, const Tensor& t, int axis, bool keepAxis = false);
Tensor softmax(const Tensor& t, const Tensor* mask = nullptr);
Tensor logSoftmax(const Tensor& t, const Tensor* mask = nullptr);

// --- kernels writing into preallocated outputs (tensor.h:116-145)
void matmulInto(Tensor& c, const Tensor& a, const Tensor& b, bool transA, bool transB,
                Real alpha = 1, Real beta = 0);
void ewiseBinaryInto(Tensor& out, EwiseOp op, const Tensor& a, const Tensor& b);
void ewiseUnaryInto(Tensor& out, EwiseOp op, const Tensor& a);
void reduceInto(Tensor& out, ReduceOp op, const Tensor& t, int axis, bool keepAxis);
void softmaxInto(Tensor& out, const Tensor& t, const Tensor* mask, bool logMode);
void accumulateReduced(Tensor& out, const Tensor& src);
void axpy(Tensor& out, const Tensor& a, Real alpha = 1);
void gatherRowsInto(Tensor& out, const Tensor& src, const std::vector<int64_t>& rows);
void scatterAddRows(Tensor& out, const Tensor& src, const std::vector<int64_t>& rows);
void transposeInto(Tensor& out, const Tensor& src, const std::vector<int>& perm);
void concatInto(Tensor& out, const std::vector<const Tensor*>& parts, int axis);
void sliceInto(Tensor& out, const Tensor& src, int axis, int64_t start, int64_t len);
void layerNormInto(Tensor& out, const Tensor& x, const Tensor& gain, const Tensor& bias,
                   Real eps, Tensor& invStd, Tensor& xhat);
void layerNormBackward(const Tensor& dy, const Tensor& gain, const Tensor& invStd,
                       const Tensor& xhat, Tensor& dx, Tensor& dgain, Tensor& dbias);

}  // namespace mtk
