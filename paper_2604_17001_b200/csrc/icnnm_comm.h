// Cross-process exchange for the H-sharded solve (one process per GPU).
// NCCL over NVLink/NVSwitch: halo shifts between ring neighbours and an
// in-place sum all-reduce of the per-iteration reduction buffer.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>

namespace icnnm_host {

class Comm {
 public:
  virtual ~Comm() = default;
  // send n floats to rank+1, receive n floats from rank-1 (periodic ring)
  virtual void shift_forward(const float* send, float* recv, size_t n, cudaStream_t s) = 0;
  // send n floats to rank-1, receive n floats from rank+1
  virtual void shift_backward(const float* send, float* recv, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_max(double* buf, size_t n, cudaStream_t s) = 0;
};

void comm_unique_id(char* out128);
std::unique_ptr<Comm> comm_create(const char* id128, int world, int rank);

}  // namespace icnnm_host
