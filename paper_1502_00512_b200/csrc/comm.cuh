// Collectives used by the multi-GPU paths.
//
//   NcclComm  -- production: one process per GPU, NCCL over NVLink/NVSwitch.
//   LocalComm -- G contexts in ONE process on one device (one host thread
//                per context), exchanging device buffers directly with a
//                host barrier + CUDA events.  Lets the data-parallel and
//                vocabulary-sharded code paths -- which are identical above
//                this interface -- run and be checked on a single B200.
// Reductions are deterministic (rank order) and leave identical results on
// every rank.
#pragma once

#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace dl {

enum class DType { F32, F64, U64, U32, BF16, U8 };

struct Comm {
  int nranks = 1, rank = 0;
  virtual ~Comm() = default;
  // in place: buf = sum over ranks (identical on all ranks)
  virtual void allreduce_sum(void* buf, size_t n, DType t, cudaStream_t st) = 0;
  // recv[r*n .. r*n+n) = rank r's send[0..n)
  virtual void allgather(const void* send, void* recv, size_t n, DType t, cudaStream_t st) = 0;
  // recv[0..n) = sum over ranks of their send[rank*n .. rank*n+n)
  virtual void reduce_scatter_sum(const void* send, void* recv, size_t n, DType t,
                                  cudaStream_t st) = 0;
  // true when other ranks' kernels run concurrently on this rank's device:
  // kernels that need the whole GPU co-resident (spin-waiting across CTAs)
  // must not be used then
  virtual bool shares_device() const { return false; }
};

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(const uint8_t id[128], int nranks, int rank);
  ~NcclComm() override;
  void allreduce_sum(void* buf, size_t n, DType t, cudaStream_t st) override;
  void allgather(const void* send, void* recv, size_t n, DType t, cudaStream_t st) override;
  void reduce_scatter_sum(const void* send, void* recv, size_t n, DType t,
                          cudaStream_t st) override;
};

struct LocalGroup {
  int G;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<const void*> ptr;
  std::vector<cudaEvent_t> ev;
  explicit LocalGroup(int g) : G(g), ptr(g), ev(g) {}
  void barrier();
};

struct LocalComm : Comm {
  LocalGroup* group;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  LocalComm(LocalGroup* g, int rank);
  ~LocalComm() override;
  void allreduce_sum(void* buf, size_t n, DType t, cudaStream_t st) override;
  void allgather(const void* send, void* recv, size_t n, DType t, cudaStream_t st) override;
  void reduce_scatter_sum(const void* send, void* recv, size_t n, DType t,
                          cudaStream_t st) override;
  bool shares_device() const override { return true; }

 private:
  void publish(const void* p, cudaStream_t st);  // ptr + ready event, then barrier + wait all
};

size_t dtype_size(DType t);

}  // namespace dl
