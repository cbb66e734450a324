// Reductions for the row-sharded RSVD: A is split by rows over
// P ranks; the only exchanges are sum all-reduces of the m-side Grams
// (l x l) and of the A^T Q panels (n x l).
//
//   NcclReducer  : ncclAllReduce(sum, float64) on the caller's stream, NCCL
//                  resolved with dlopen("libnccl.so.2") (torch's bundled copy or
//                  the system one) — one process per GPU over NVLink/NVSwitch.
//   GroupReducer : in-process ranks (one host thread + handle each) on devices
//                  of one process; host barriers only, never a device-side
//                  wait, so P ranks can share one GPU safely.  The sum is formed
//                  by rank 0 in fixed rank order (deterministic).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace rsvd {
namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.getErrorString =
        reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy &&
             api.getErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks the required symbols";
  });
  if (!api.ok) throw CudaError("NCCL unavailable: " + api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().getErrorString(r));
}

struct NcclReducer final : Reducer {
  ncclComm_t comm = nullptr;
  NcclReducer(int nranks, int rank, const unsigned char* id) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().commInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclReducer() override {
    if (comm) nccl().commDestroy(comm);
  }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t st) override {
    nccl_check(nccl().allReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, comm,
                                st),
               "ncclAllReduce");
  }
  bool capturable() const override { return true; }
};

// --------------------------------------------------------------- in-process
constexpr int kMaxGroup = 16;
struct SlotPtrs {
  const double* p[kMaxGroup];
};

__global__ void group_sum_kernel(SlotPtrs s, int n, int64_t count, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    for (int r = 0; r < n; ++r) v += s.p[r][e];
    out[e] = v;
  }
}

}  // namespace

struct Group {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<double*> slots;
  double* sum = nullptr;
  int64_t cap = 0;
  explicit Group(int nranks) : n(nranks), slots(nranks, nullptr) {}
  ~Group() {
    if (sum) cudaFree(sum);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {
struct GroupReducer final : Reducer {
  Group* g;
  int rank;
  GroupReducer(Group* grp, int r) : g(grp), rank(r) {}
  void allreduce_sum(double* buf, int64_t count, cudaStream_t st) override {
    RSVD_CUDA(cudaStreamSynchronize(st));
    g->slots[rank] = buf;
    g->barrier();  // every rank's contribution is complete
    if (rank == 0) {
      if (g->cap < count) {
        if (g->sum) RSVD_CUDA(cudaFree(g->sum));
        RSVD_CUDA(cudaMalloc(&g->sum, sizeof(double) * count));
        g->cap = count;
      }
      SlotPtrs sp{};
      for (int r = 0; r < g->n; ++r) sp.p[r] = g->slots[r];
      const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(count, 256), 8 * num_sms()));
      group_sum_kernel<<<std::max(blocks, 1), 256, 0, st>>>(sp, g->n, count, g->sum);
      RSVD_LAUNCH("group_sum_kernel");
      RSVD_CUDA(cudaStreamSynchronize(st));
    }
    g->barrier();  // the sum is ready
    RSVD_CUDA(cudaMemcpyAsync(buf, g->sum, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    RSVD_CUDA(cudaStreamSynchronize(st));
    g->barrier();  // everyone copied it out before the next reduction reuses it
  }
  bool capturable() const override { return false; }
};
}  // namespace

Group* group_create(int nranks) {
  if (nranks < 1 || nranks > kMaxGroup) throw CudaError("group size must be in [1, 16]");
  return new Group(nranks);
}
void group_destroy(Group* g) { delete g; }
std::unique_ptr<Reducer> make_group_reducer(Group* g, int rank) {
  if (!g || rank < 0 || rank >= g->n) throw CudaError("bad group rank");
  return std::make_unique<GroupReducer>(g, rank);
}
std::unique_ptr<Reducer> make_nccl_reducer(int nranks, int rank, const unsigned char* id) {
  return std::make_unique<NcclReducer>(nranks, rank, id);
}
void nccl_unique_id(unsigned char* out) {
  ncclUniqueId uid;
  nccl_check(nccl().getUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

}  // namespace rsvd
