// Device context and error mapping for the host framework.
#include "mtk/device.h"

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace mtk {

namespace {
int g_selected = -1;
}

void mtkcCheck(int rc, const char* what) {
  if(rc == MTKC_OK)
    return;
  std::string msg = std::string(mtkc_last_error()) + " [" + what + "]";
  switch(rc) {
    case MTKC_DIMENSION: throw DimensionError(msg);
    case MTKC_NUMERIC: throw NumericError(msg);
    case MTKC_CONTRACT: throw ContractError(msg);
    case MTKC_DATA: throw DataError(msg);
    default: throw Error("device error: " + msg);
  }
}

void Device::selectDevice(int index) { g_selected = index; }

Device::Device() {
  index_ = g_selected;
  if(index_ < 0) {
    const char* e = std::getenv("LOCAL_RANK");
    index_ = e ? std::atoi(e) : 0;
    int n = 0;
    if(mtkc_device_count(&n) == MTKC_OK && n > 0)
      index_ %= n;
  }
  MTKC(mtkc_init(index_));
  MTKC(mtkc_stream_create(&stream_));
  MTKC(mtkc_stream_create(&comm_));
  void* f = nullptr;
  MTKC(mtkc_malloc(&f, 256));
  flags_ = (int*)f;
  MTKC(mtkc_memset(flags_, 0, 256, stream_));
  MTKC(mtkc_sm_count(&sms_));
  const char* p = std::getenv("MTK_PRECISION");
  if(p && (std::string(p) == "fp32" || std::string(p) == "FP32"))
    precision_ = Precision::FP32;
  if(const char* r = std::getenv("MTK_DROPOUT_RNG")) {
    const std::string v(r);
    dropoutRng_ = v == "host" ? DropoutRng::Host : v == "device" ? DropoutRng::Device
                                                                : DropoutRng::Auto;
  }
}

Device& Device::get() {
  static Device* d = new Device();  // intentionally leaked: lives for the process
  return *d;
}

float* Device::scratch(size_t bytes) {
  if(bytes <= scratchBytes_ && scratch_)
    return scratch_->ptr;
  // generous first reservation (HBM is plentiful; a regrow costs a stream
  // sync + cudaMalloc, tens of milliseconds on a fresh process), then double
  size_t want = std::max(std::max(bytes, (size_t)1 << 30), 2 * scratchBytes_);
  sync();
  scratch_ = std::make_shared<DeviceBuffer>(want / sizeof(float));
  scratchBytes_ = want;
  return scratch_->ptr;
}

void Device::sync() { MTKC(mtkc_stream_sync(stream_)); }

void* Device::sideStream() {
  if(!side_) {
    MTKC(mtkc_stream_create(&side_));
    MTKC(mtkc_event_create(&forkEv_));
    MTKC(mtkc_event_create(&joinEv_));
  }
  return side_;
}

void Device::forkSide() {
  sideStream();
  MTKC(mtkc_event_record(forkEv_, stream_));
  MTKC(mtkc_stream_wait_event(side_, forkEv_));
}

void Device::joinSide() {
  MTKC(mtkc_event_record(joinEv_, side_));
  MTKC(mtkc_stream_wait_event(stream_, joinEv_));
}

void Device::upload(void* dst, const void* src, size_t bytes) {
  if(!bytes)
    return;
  size_t need = (bytes + 255) & ~(size_t)255;
  // Default: a plain cudaMemcpyAsync from the caller's (pageable) buffer.
  // The driver takes the bytes before returning and carries small copies
  // inline in the stream's command buffer, which measured faster than the
  // pinned staging ring below, both with a DMA copy (base 772k vs 795k
  // words/s) and with the PDL copy kernel reading mapped host memory (783k;
  // tiny 1.37M vs 1.48M).  MTK_UPLOAD_RING=1 selects the ring.
  static const bool ring = getenv("MTK_UPLOAD_RING") && getenv("MTK_UPLOAD_RING")[0] == '1';
  if(!ring) {
    MTKC(mtkc_memcpy_h2d(dst, src, bytes, stream_));
    return;
  }
  if(!pinned_) {
    pinnedBytes_ = (size_t)64 << 20;
    void* p = nullptr;
    MTKC(mtkc_host_alloc_pinned(&p, pinnedBytes_));
    pinned_ = (char*)p;
  }
  if(need > pinnedBytes_ / 2) {  // oversized: plain (possibly blocking) copy
    MTKC(mtkc_memcpy_h2d(dst, src, bytes, stream_));
    return;
  }
  if(head_ + need > pinnedBytes_)
    head_ = 0;
  size_t b = head_, e = head_ + need;
  // wait for earlier copies still reading the region we are about to reuse
  for(size_t i = 0; i < inflight_.size();) {
    Pending& q = inflight_[i];
    if(q.begin < e && b < q.end) {
      MTKC(mtkc_event_sync(q.event));  // host waits for that copy only
      eventPool_.push_back(q.event);
      inflight_.erase(inflight_.begin() + (long)i);
    } else {
      ++i;
    }
  }
  std::memcpy(pinned_ + b, src, bytes);
  MTKC(mtkc_upload_pinned(dst, pinned_ + b, bytes, stream_));
  void* ev = nullptr;
  if(!eventPool_.empty()) {
    ev = eventPool_.back();
    eventPool_.pop_back();
  } else {
    MTKC(mtkc_event_create(&ev));
  }
  MTKC(mtkc_event_record(ev, stream_));
  inflight_.push_back(Pending{b, e, ev});
  head_ = e;
}

void Device::checkFlags(const std::string& where) {
  int host = 0;
  MTKC(mtkc_memcpy_d2h(&host, flags_, sizeof(int), stream_));
  sync();
  if(!host)
    return;
  MTKC(mtkc_memset(flags_, 0, sizeof(int), stream_));
  if(host & MTKC_FLAG_MASKED_ROW)
    throw NumericError("softmax over a fully-masked row (" + where + ")");
  if(host & MTKC_FLAG_DIV_ZERO)
    throw NumericError("division by zero in elementwise div (" + where + ")");
  if(host & MTKC_FLAG_BAD_ID)
    throw DataError("row/token id out of range (" + where + ")");
  if(host & MTKC_FLAG_NONFINITE)
    throw NumericError("non-finite value (" + where + ")");
}

}  // namespace mtk
