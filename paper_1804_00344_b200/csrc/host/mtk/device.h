// Per-process device context: the compute stream every kernel is issued on,
// the communication stream, the device error-flag word and a shared
// stream-ordered scratch buffer (split-K partials, column-sum partials).
#pragma once

#include <cstddef>
#include <memory>
#include <string>
#include <vector>

#include "mtk/tensor.h"
#include "mtk_cuda.h"

namespace mtk {

// GEMM arithmetic.  FP32 = CUDA-core kernel with the reference's exact
// summation order (parity mode); TF32 = tcgen05 tensor cores (default).
enum class Precision { FP32 = 0, TF32 = 1 };

// Where dropout masks come from.  Host = the reference's own draws (the
// graph's mt19937_64, graph.cpp:817-830; bit-exact, uploaded as constants);
// Device = counter-based Philox masks recomputed inside the kernels (never
// stored or uploaded; keyed by one draw of the same graph RNG).  Auto = Host
// in FP32 (parity) mode, Device in TF32 (throughput) mode.
enum class DropoutRng { Auto = 0, Host = 1, Device = 2 };

class Device {
public:
  static Device& get();  // initialises the device on first use

  void* stream() const { return stream_; }
  void* commStream() const { return comm_; }
  int* flags() const { return flags_; }
  int sms() const { return sms_; }
  int index() const { return index_; }
  Precision precision() const { return precision_; }
  void setPrecision(Precision p) { precision_ = p; }
  DropoutRng dropoutRng() const { return dropoutRng_; }
  void setDropoutRng(DropoutRng r) { dropoutRng_ = r; }
  bool deviceDropout() const {
    return dropoutRng_ == DropoutRng::Device ||
           (dropoutRng_ == DropoutRng::Auto && precision_ == Precision::TF32);
  }

  float* scratch(size_t bytes);  // stream-ordered scratch, grows on demand
  // Second compute stream for independent work inside one op (the two
  // directions of the bidirectional RNN encoder): forkSide() makes it wait
  // for the compute stream, joinSide() makes the compute stream wait for it.
  void* sideStream();
  void forkSide();
  void joinSide();
  size_t scratchBytes() const { return scratchBytes_; }

  // Asynchronous host->device copy on the compute stream through a pinned
  // staging ring (a pageable cudaMemcpyAsync may block the host until the
  // stream drains, which would serialise graph building with the GPU).
  void upload(void* dst, const void* src, size_t bytes);

  void sync();        // synchronise the compute stream
  // synchronise, read and clear the flag word, throw the mapped error
  void checkFlags(const std::string& where);
  static void selectDevice(int index);  // before first get()

private:
  Device();
  void* stream_ = nullptr;
  void* comm_ = nullptr;
  int* flags_ = nullptr;
  int sms_ = 148;
  int index_ = 0;
  Precision precision_ = Precision::TF32;
  DropoutRng dropoutRng_ = DropoutRng::Auto;
  std::shared_ptr<DeviceBuffer> scratch_;
  void* side_ = nullptr;
  void* forkEv_ = nullptr;
  void* joinEv_ = nullptr;
  size_t scratchBytes_ = 0;
  // pinned staging ring
  struct Pending {
    size_t begin, end;
    void* event;
  };
  char* pinned_ = nullptr;
  size_t pinnedBytes_ = 0, head_ = 0;
  std::vector<Pending> inflight_;
  std::vector<void*> eventPool_;
};

// Map an mtkc status code to the reference's exception types.
void mtkcCheck(int rc, const char* what);
#define MTKC(call) ::mtk::mtkcCheck((call), #call)

}  // namespace mtk
