// ensei_b200.hpp -- header-only C++ host mirror of the REF operator surface over the
// C ABI (include/ensei_gpu.h).  Same names / argument meaning / exception types as
// REF (namespace ensei -> ensei_b200), batched where REF works one block at a time.
// Link: -lensei_gpu (paper_2003_05328_b200/libensei_gpu.so) -lcudart.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/ensei_gpu.h"

namespace ensei_b200 {

// REF errors.hpp:7-37, thrown from the C status codes
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct OrderNotDividing : Error { using Error::Error; };
struct SearchExhausted : Error { using Error::Error; };
struct BadRoot : Error { using Error::Error; };
struct BadGeometry : Error { using Error::Error; };
struct GeometryMismatch : Error { using Error::Error; };
struct DomainMismatch : Error { using Error::Error; };
struct NoiseExhausted : Error { using Error::Error; };
struct ChainViolation : Error { using Error::Error; };
struct LengthMismatch : Error { using Error::Error; };
struct RangeViolation : Error { using Error::Error; };
struct ProtocolOrderViolation : Error { using Error::Error; };
struct RangeOverflow : Error { using Error::Error; };
struct MalformedPayload : Error { using Error::Error; };
struct TransportError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(int rc) {
  if (rc == ENSEI_OK) return;
  std::string m = ensei_gpu_last_error();
  switch (rc) {
    case ENSEI_ERR_ORDER_NOT_DIVIDING: throw OrderNotDividing(m);
    case ENSEI_ERR_SEARCH_EXHAUSTED: throw SearchExhausted(m);
    case ENSEI_ERR_BAD_ROOT: throw BadRoot(m);
    case ENSEI_ERR_BAD_GEOMETRY: throw BadGeometry(m);
    case ENSEI_ERR_GEOMETRY_MISMATCH: throw GeometryMismatch(m);
    case ENSEI_ERR_DOMAIN_MISMATCH: throw DomainMismatch(m);
    case ENSEI_ERR_NOISE_EXHAUSTED: throw NoiseExhausted(m);
    case ENSEI_ERR_CHAIN_VIOLATION: throw ChainViolation(m);
    case ENSEI_ERR_LENGTH_MISMATCH: throw LengthMismatch(m);
    case ENSEI_ERR_RANGE_VIOLATION: throw RangeViolation(m);
    case ENSEI_ERR_PROTOCOL_ORDER: throw ProtocolOrderViolation(m);
    case ENSEI_ERR_RANGE_OVERFLOW: throw RangeOverflow(m);
    case ENSEI_ERR_MALFORMED_PAYLOAD: throw MalformedPayload(m);
    case ENSEI_ERR_TRANSPORT: throw TransportError(m);
    case ENSEI_ERR_CUDA: case ENSEI_ERR_UNSUPPORTED: case ENSEI_ERR_INVALID_ARGUMENT: throw DeviceError(m);
    default: throw Error(m);
  }
}

template <class T>
struct DeviceBuffer {
  T* p = nullptr;
  size_t n = 0;
  explicit DeviceBuffer(size_t count) : n(count) {
    if (count && cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) throw DeviceError("cudaMalloc failed");
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { if (p) cudaFree(p); }
  void upload(const T* h, size_t count) { cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice); }
  void download(T* h, size_t count) const { cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost); }
};

// RlweParams + ModulusChain::unified on one device (REF ringbfv.cpp:65-87)
class Context {
 public:
  Context(uint32_t n, std::vector<uint64_t> q, uint64_t p, int device = 0) : n_(n) {
    check(ensei_gpu_ctx_create(device, n, q.data(), (uint32_t)q.size(), p, &h_));
  }
  ~Context() { ensei_gpu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ensei_gpu_ctx* get() const { return h_; }
  uint32_t n() const { return n_; }

  // NegacyclicPlan::forward / inverse (REF ringbfv.cpp:49-59) on `polys` = k*n
  // residues mod q_i (natural order both sides, REF layout).
  void negacyclic_forward(std::vector<uint64_t>& polys, uint32_t prime = 0) const { transform(polys, prime, 0); }
  void negacyclic_inverse(std::vector<uint64_t>& polys, uint32_t prime = 0) const { transform(polys, prime, 1); }
  // encode_slots / decode_slots (REF ringbfv.cpp:109-125)
  void encode_slots(std::vector<uint64_t>& v) const { transform(v, ENSEI_MOD_P, 1); }
  void decode_slots(std::vector<uint64_t>& v) const { transform(v, ENSEI_MOD_P, 0); }
  // ntt_2d / intt_2d (REF ntt.cpp:139-153) on k rows x cols tiles
  void ntt_2d(std::vector<uint64_t>& tiles, uint32_t rows, uint32_t cols, bool inverse = false) const {
    DeviceBuffer<uint64_t> d(tiles.size());
    d.upload(tiles.data(), tiles.size());
    check(ensei_gpu_ntt2d(h_, inverse ? 1 : 0, rows, cols, d.p, tiles.size() / ((size_t)rows * cols), nullptr));
    d.download(tiles.data(), tiles.size());
  }

 private:
  void transform(std::vector<uint64_t>& v, uint32_t modulus, int inverse) const {
    if (v.size() % n_) throw LengthMismatch("vector length must be a multiple of n");
    DeviceBuffer<uint64_t> d(v.size());
    d.upload(v.data(), v.size());
    check(ensei_gpu_negacyclic(h_, modulus, inverse, ENSEI_LAYOUT_NATURAL, d.p, v.size() / n_, nullptr));
    d.download(v.data(), v.size());
  }
  ensei_gpu_ctx* h_ = nullptr;
  uint32_t n_;
};

}  // namespace ensei_b200
