// Collectives of the multi-GPU evaluation: one process per
// GPU, the exchanges between the upward and downward passes carried out by
// NCCL over NVLink / NVSwitch inside libkafmm (kafmm_get_unique_id,
// kafmm_setup_dist).  NCCL is opened at run time (dlopen "libnccl.so.2"):
// inside a process that already loaded torch this is torch's NCCL, and a
// single-GPU user of the library never needs it.
//
// A second implementation, LocalComm, runs the ranks of one group as host
// threads of a single process (kafmm_comm_local_create): a host barrier plus
// device-to-device copies on each rank's stream.  It exists so that the
// partitioned evaluation can be checked on one GPU (tests/test_gpu_dist.py);
// ranks never wait on each other on the device, only on the host.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kafmm_internal.h"

namespace kafmm {

// ---------------------------------------------------------------------------
// NCCL through dlopen
// ---------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.err = std::string("cannot open libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        a.err = std::string("libnccl.so.2 lacks ") + name;
      }
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    return a;
  }();
  if (!api.ok) throw Error{KAFMM_ENCCL, api.err};
  return api;
}

#define KF_NCCL(call)                                                                                      \
  do {                                                                                                     \
    ncclResult_t r_ = (call);                                                                              \
    if (r_ != ncclSuccess) throw ::kafmm::Error{KAFMM_ENCCL, std::string(#call) + ": " + api.GetErrorString(r_)}; \
  } while (0)

void nccl_unique_id(unsigned char id[128]) {
  const NcclApi& api = nccl();
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  KF_NCCL(api.GetUniqueId(&u));
  std::memcpy(id, &u, 128);
}

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  NcclComm(const unsigned char id[128], int r, int w) {
    const NcclApi& api = nccl();
    rank = r;
    world = w;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    KF_NCCL(api.CommInitRank(&c, w, u, r));
  }
  ~NcclComm() override {
    if (c) nccl().CommDestroy(c);
  }
  void alltoallv(const double* sbuf, const int64_t* sdispl, const int64_t* scount, double* rbuf,
                 const int64_t* rdispl, const int64_t* rcount, cudaStream_t s) override {
    const NcclApi& api = nccl();
    KF_NCCL(api.GroupStart());
    for (int q = 0; q < world; ++q) {
      if (scount[q] > 0) KF_NCCL(api.Send(sbuf + sdispl[q], (size_t)scount[q], ncclFloat64, q, c, s));
      if (rcount[q] > 0) KF_NCCL(api.Recv(rbuf + rdispl[q], (size_t)rcount[q], ncclFloat64, q, c, s));
    }
    KF_NCCL(api.GroupEnd());
  }
  void allreduce(double* buf, int64_t count, cudaStream_t s) override {
    if (count <= 0) return;
    const NcclApi& api = nccl();
    KF_NCCL(api.AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, c, s));
  }
  const char* kind() const override { return "nccl"; }
};

Comm* make_nccl_comm(const unsigned char id[128], int rank, int world) { return new NcclComm(id, rank, world); }

// ---------------------------------------------------------------------------
// in-process group (test transport)
// ---------------------------------------------------------------------------
struct LocalGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  int refs = 0;
  struct Slot {
    const double* sbuf = nullptr;
    const int64_t* sdispl = nullptr;
    const int64_t* scount = nullptr;
    const double* buf = nullptr;
  };
  std::vector<Slot> slot;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

__global__ void k_sum_into(double* __restrict__ out, const double* __restrict__ a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] += a[i];
}

struct LocalComm : Comm {
  LocalGroup* g;
  LocalComm(LocalGroup* grp, int r) : g(grp) {
    rank = r;
    world = grp->world;
  }
  ~LocalComm() override {
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) delete g;
  }
  void alltoallv(const double* sbuf, const int64_t* sdispl, const int64_t* scount, double* rbuf,
                 const int64_t* rdispl, const int64_t* rcount, cudaStream_t s) override {
    KF_CUDA(cudaStreamSynchronize(s));  // the send buffer is complete
    g->slot[rank] = {sbuf, sdispl, scount, nullptr};
    g->barrier();
    for (int q = 0; q < world; ++q) {
      const LocalGroup::Slot& o = g->slot[q];
      if (o.scount[rank] != rcount[q])
        throw Error{KAFMM_ENCCL, "local alltoallv: send / receive counts disagree"};
      if (rcount[q] > 0)
        KF_CUDA(cudaMemcpyAsync(rbuf + rdispl[q], o.sbuf + o.sdispl[rank], (size_t)rcount[q] * 8,
                                cudaMemcpyDeviceToDevice, s));
    }
    KF_CUDA(cudaStreamSynchronize(s));
    g->barrier();  // every receiver has copied: the senders may reuse their buffers
  }
  void allreduce(double* buf, int64_t count, cudaStream_t s) override {
    if (count <= 0) return;
    KF_CUDA(cudaStreamSynchronize(s));
    g->slot[rank].buf = buf;
    double* tmp = nullptr;
    KF_CUDA(cudaMalloc(&tmp, (size_t)count * 8));
    KF_CUDA(cudaMemsetAsync(tmp, 0, (size_t)count * 8, s));
    g->barrier();
    for (int q = 0; q < world; ++q) {  // the same summation order on every rank
      k_sum_into<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(tmp, g->slot[q].buf, count);
      KF_CHECK_LAUNCH();
    }
    KF_CUDA(cudaStreamSynchronize(s));
    g->barrier();  // everyone has read every buffer
    KF_CUDA(cudaMemcpyAsync(buf, tmp, (size_t)count * 8, cudaMemcpyDeviceToDevice, s));
    KF_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
  }
  const char* kind() const override { return "local"; }
};

void make_local_comms(int world, Comm** out) {
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->refs = world;
  g->slot.resize(world);
  for (int r = 0; r < world; ++r) out[r] = new LocalComm(g, r);
}

// all-gather of one int64 per rank through alltoallv (setup only)
std::vector<int64_t> Comm::allgather_count(int64_t mine, cudaStream_t s) {
  std::vector<int64_t> sd(world, 0), sc(world, 1), rd(world), rc(world, 1);
  for (int q = 0; q < world; ++q) rd[q] = q;
  double *d_in = nullptr, *d_out = nullptr;
  KF_CUDA(cudaMalloc(&d_in, 8));
  KF_CUDA(cudaMalloc(&d_out, 8 * world));
  const double v = (double)mine;  // counts < 2^31: exact in a double
  KF_CUDA(cudaMemcpyAsync(d_in, &v, 8, cudaMemcpyHostToDevice, s));
  alltoallv(d_in, sd.data(), sc.data(), d_out, rd.data(), rc.data(), s);
  std::vector<double> h(world);
  KF_CUDA(cudaMemcpyAsync(h.data(), d_out, 8 * world, cudaMemcpyDeviceToHost, s));
  KF_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_in);
  cudaFree(d_out);
  std::vector<int64_t> out(world);
  for (int q = 0; q < world; ++q) out[q] = (int64_t)h[q];
  return out;
}

}  // namespace kafmm
