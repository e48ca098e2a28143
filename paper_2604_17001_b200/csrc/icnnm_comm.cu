// NCCL implementation of the sharded-solve exchange (icnnm_comm.h).
#include <nccl.h>

#include <cstring>
#include <string>

#include "../../include/icnnm_b200.h"
#include "icnnm_comm.h"

namespace icnnm_host {

struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);

#define NK(x)                                                                          \
  do {                                                                                 \
    ncclResult_t r_ = (x);                                                             \
    if (r_ != ncclSuccess)                                                             \
      ::icnnm_host::fail(ICNNM_CUDA_ERROR, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

class NcclComm final : public Comm {
 public:
  NcclComm(const char* id128, int world, int rank) : world_(world), rank_(rank) {
    ncclUniqueId id;
    static_assert(sizeof(id.internal) == ICNNM_NCCL_UNIQUE_ID_BYTES, "nccl id size");
    std::memcpy(id.internal, id128, sizeof(id.internal));
    NK(ncclCommInitRank(&comm_, world, id, rank));
  }
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  void shift_forward(const float* send, float* recv, size_t n, cudaStream_t s) override {
    const int next = (rank_ + 1) % world_, prev = (rank_ + world_ - 1) % world_;
    NK(ncclGroupStart());
    NK(ncclSend(send, n, ncclFloat32, next, comm_, s));
    NK(ncclRecv(recv, n, ncclFloat32, prev, comm_, s));
    NK(ncclGroupEnd());
  }
  void shift_backward(const float* send, float* recv, size_t n, cudaStream_t s) override {
    const int next = (rank_ + 1) % world_, prev = (rank_ + world_ - 1) % world_;
    NK(ncclGroupStart());
    NK(ncclSend(send, n, ncclFloat32, prev, comm_, s));
    NK(ncclRecv(recv, n, ncclFloat32, next, comm_, s));
    NK(ncclGroupEnd());
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override {
    NK(ncclAllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, s));
  }
  void allreduce_max(double* buf, size_t n, cudaStream_t s) override {
    NK(ncclAllReduce(buf, buf, n, ncclFloat64, ncclMax, comm_, s));
  }

 private:
  ncclComm_t comm_ = nullptr;
  int world_, rank_;
};

void comm_unique_id(char* out128) {
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  std::memcpy(out128, id.internal, sizeof(id.internal));
}

std::unique_ptr<Comm> comm_create(const char* id128, int world, int rank) {
  return std::make_unique<NcclComm>(id128, world, rank);
}

}  // namespace icnnm_host
