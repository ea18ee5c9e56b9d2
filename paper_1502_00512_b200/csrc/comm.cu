// Collectives for the multi-GPU paths (comm.cuh).
#include <cstring>

#include "comm.cuh"

namespace dl {

size_t dtype_size(DType t) {
  switch (t) {
    case DType::F32: return 4;
    case DType::U32: return 4;
    case DType::F64: return 8;
    case DType::U64: return 8;
    case DType::BF16: return 2;
    case DType::U8: return 1;
  }
  return 4;
}

static ncclDataType_t nccl_type(DType t) {
  switch (t) {
    case DType::F32: return ncclFloat;
    case DType::F64: return ncclDouble;
    case DType::U64: return ncclUint64;
    case DType::U32: return ncclUint32;
    case DType::BF16: return ncclBfloat16;
    case DType::U8: return ncclUint8;
  }
  return ncclFloat;
}

static void nccl_ok(ncclResult_t r, const char* op = "", size_t n = 0, DType t = DType::F32) {
  if (r != ncclSuccess)
    throw Error(3, std::string("NCCL: ") + ncclGetErrorString(r) + " (" + op + ", " +
                       std::to_string(n) + " x " + std::to_string(dtype_size(t)) + " B)");
}

NcclComm::NcclComm(const uint8_t id[128], int n, int r) {
  nranks = n;
  rank = r;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  nccl_ok(ncclCommInitRank(&comm, n, u, r));
}

NcclComm::~NcclComm() {
  if (comm) ncclCommDestroy(comm);
}

void NcclComm::allreduce_sum(void* buf, size_t n, DType t, cudaStream_t st) {
  nccl_ok(ncclAllReduce(buf, buf, n, nccl_type(t), ncclSum, comm, st), "allreduce", n, t);
}

void NcclComm::allgather(const void* send, void* recv, size_t n, DType t, cudaStream_t st) {
  nccl_ok(ncclAllGather(send, recv, n, nccl_type(t), comm, st), "allgather", n, t);
}

void NcclComm::reduce_scatter_sum(const void* send, void* recv, size_t n, DType t,
                                  cudaStream_t st) {
  nccl_ok(ncclReduceScatter(send, recv, n, nccl_type(t), ncclSum, comm, st), "reduce_scatter",
          n, t);
}

// ------------------------------------------------------------- LocalComm
void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(m);
  const long gen = generation;
  if (++arrived == G) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != gen; });
  }
}

LocalComm::LocalComm(LocalGroup* g, int r) : group(g) {
  nranks = g->G;
  rank = r;
  DL_CUDA(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
  DL_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
}

LocalComm::~LocalComm() {
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  if (tmp) cudaFree(tmp);
}

void LocalComm::publish(const void* p, cudaStream_t st) {
  DL_CUDA(cudaEventRecord(ev_a, st));
  group->ptr[rank] = p;
  group->ev[rank] = ev_a;
  group->barrier();
  for (int r = 0; r < nranks; ++r) DL_CUDA(cudaStreamWaitEvent(st, group->ev[r], 0));
}

namespace {
struct Ptrs {
  const void* p[16];
};

// bf16: summed in fp32 in rank order, rounded once
__global__ void k_sum_ranks_bf16(bf16* out, Ptrs in, int G, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float s = __bfloat162float(static_cast<const bf16*>(in.p[0])[i]);
    for (int r = 1; r < G; ++r) s += __bfloat162float(static_cast<const bf16*>(in.p[r])[i]);
    out[i] = __float2bfloat16_rn(s);
  }
}

template <class T>
__global__ void k_sum_ranks(T* out, Ptrs in, int G, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    T s = static_cast<const T*>(in.p[0])[i];
    for (int r = 1; r < G; ++r) s += static_cast<const T*>(in.p[r])[i];
    out[i] = s;
  }
}
}  // namespace

void LocalComm::allreduce_sum(void* buf, size_t n, DType t, cudaStream_t st) {
  DL_REQUIRE(nranks <= 16, 1, "LocalComm: at most 16 ranks");
  const size_t bytes = n * dtype_size(t);
  if (bytes > tmp_bytes) {
    if (tmp) cudaFree(tmp);
    DL_CUDA(cudaMalloc(&tmp, bytes));
    tmp_bytes = bytes;
  }
  publish(buf, st);
  Ptrs ps{};
  for (int r = 0; r < nranks; ++r) ps.p[r] = group->ptr[r];
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
  if (n > 0) {
    switch (t) {
      case DType::F32: k_sum_ranks<float><<<grid, 256, 0, st>>>((float*)tmp, ps, nranks, n); break;
      case DType::F64: k_sum_ranks<double><<<grid, 256, 0, st>>>((double*)tmp, ps, nranks, n); break;
      case DType::U64:
        k_sum_ranks<unsigned long long><<<grid, 256, 0, st>>>((unsigned long long*)tmp, ps, nranks, n);
        break;
      case DType::U32: k_sum_ranks<unsigned><<<grid, 256, 0, st>>>((unsigned*)tmp, ps, nranks, n); break;
      case DType::BF16: k_sum_ranks_bf16<<<grid, 256, 0, st>>>((bf16*)tmp, ps, nranks, n); break;
    }
    DL_CUDA(cudaGetLastError());
  }
  // every rank has read every buffer before anyone overwrites its own
  DL_CUDA(cudaEventRecord(ev_b, st));
  group->barrier();
  group->ev[rank] = ev_b;
  group->barrier();
  for (int r = 0; r < nranks; ++r) DL_CUDA(cudaStreamWaitEvent(st, group->ev[r], 0));
  group->barrier();
  if (bytes) DL_CUDA(cudaMemcpyAsync(buf, tmp, bytes, cudaMemcpyDeviceToDevice, st));
}

void LocalComm::reduce_scatter_sum(const void* send, void* recv, size_t n, DType t,
                                   cudaStream_t st) {
  DL_REQUIRE(nranks <= 16, 1, "LocalComm: at most 16 ranks");
  DL_REQUIRE(t == DType::F32, 1, "LocalComm: reduce_scatter supports f32");
  publish(send, st);
  Ptrs ps{};
  for (int r = 0; r < nranks; ++r)
    ps.p[r] = static_cast<const float*>(group->ptr[r]) + (size_t)rank * n;
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
  if (n > 0) {
    k_sum_ranks<float><<<grid, 256, 0, st>>>(static_cast<float*>(recv), ps, nranks, n);
    DL_CUDA(cudaGetLastError());
  }
  // every rank has read every buffer before anyone reuses its own
  DL_CUDA(cudaEventRecord(ev_b, st));
  group->barrier();
  group->ev[rank] = ev_b;
  group->barrier();
  for (int r = 0; r < nranks; ++r) DL_CUDA(cudaStreamWaitEvent(st, group->ev[r], 0));
  group->barrier();
}

void LocalComm::allgather(const void* send, void* recv, size_t n, DType t, cudaStream_t st) {
  const size_t bytes = n * dtype_size(t);
  publish(send, st);
  for (int r = 0; r < nranks; ++r)
    if (bytes)
      DL_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + r * bytes, group->ptr[r], bytes,
                              cudaMemcpyDeviceToDevice, st));
  DL_CUDA(cudaEventRecord(ev_b, st));
  group->barrier();
  group->ev[rank] = ev_b;
  group->barrier();
  for (int r = 0; r < nranks; ++r) DL_CUDA(cudaStreamWaitEvent(st, group->ev[r], 0));
  group->barrier();
}

}  // namespace dl
