// comm.cu -- transports of the multi-GPU slab solvers (comm.h).
//  * NCCL (one process per GPU): grouped ncclSend/ncclRecv of whole rows or
//    planes, in-place ncclAllGather, ncclAllReduce; libnccl.so.2 (the one
//    torch ships) is loaded at run time, so a single-GPU build needs no NCCL.
//  * loopback: P virtual ranks in one process on one GPU; halos copied
//    device-to-device between their slabs, coarse arrays shared.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>

#include "comm.h"
#include "mg.h"

namespace {

// ------------------------------------------------------------------ NCCL
typedef struct ncclComm *ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat32 = 7, ncclFloat64 = 8, ncclUint64 = 5 };
enum { ncclSum = 0, ncclMax = 2 };

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;   // optional
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                             // optional
  bool load() {
    if (ok) return true;
    const char *names[] = {getenv("MG_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *nm : names)
      if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      why = "libnccl.so.2 not found (set MG_NCCL_LIB)";
      return false;
    }
#define SYM(f, name)                                         \
  f = reinterpret_cast<decltype(f)>(dlsym(h, name));         \
  if (!f) {                                                  \
    why = std::string("missing NCCL symbol ") + name;        \
    return false;                                            \
  }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(AllGather, "ncclAllGather");
    SYM(AllReduce, "ncclAllReduce");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    CommGetAsyncError = reinterpret_cast<decltype(CommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    CommAbort = reinterpret_cast<decltype(CommAbort)>(dlsym(h, "ncclCommAbort"));
    ok = true;
    return true;
  }
};
NcclApi &nccl() {
  static NcclApi a;
  return a;
}

}  // namespace

namespace mg {

struct LoopComm : Comm2 {
  cudaError_t exchange(const std::vector<char *> &p, size_t pb, const std::vector<int> &lo, const std::vector<int> &hi,
                       int g, cudaStream_t st) override {
    for (int i = 0; i < P; i++) {
      if (i > 0) {   // rows [lo_i - g, lo_i) are owned by rank i-1
        cudaError_t e = cudaMemcpyAsync(p[i] + (int64_t)(lo[i] - g) * pb, p[i - 1] + (int64_t)(lo[i] - g) * pb, g * pb,
                                        cudaMemcpyDeviceToDevice, st);
        if (e) return e;
      }
      if (i + 1 < P) {   // rows [hi_i, hi_i + g) are owned by rank i+1
        cudaError_t e = cudaMemcpyAsync(p[i] + (int64_t)hi[i] * pb, p[i + 1] + (int64_t)hi[i] * pb, g * pb,
                                        cudaMemcpyDeviceToDevice, st);
        if (e) return e;
      }
    }
    return cudaSuccess;
  }
  cudaError_t allgather(char *, size_t, int, int, int, cudaStream_t) override { return cudaSuccess; }
  cudaError_t allreduce_max_u64(unsigned long long *, int, cudaStream_t) override { return cudaSuccess; }
  cudaError_t allreduce_sum_f64(double *, int, cudaStream_t) override { return cudaSuccess; }
};

struct NcclComm : Comm2 {
  int q = 0;
  int dtype = ncclFloat64;
  ncclComm_t comm = nullptr;
  std::string err;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  bool init(int P_, int q_, const void *id, int esz) {
    P = P_;
    q = q_;
    dtype = esz == 8 ? ncclFloat64 : ncclFloat32;
    if (!nccl().load()) {
      err = nccl().why;
      return false;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclResult_t r = nccl().CommInitRank(&comm, P, uid, q);
    if (r != 0) {
      err = std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
      comm = nullptr;
      return false;
    }
    return true;
  }
  cudaError_t check(ncclResult_t r, const char *what) {
    if (r == 0) return cudaSuccess;
    err = std::string(what) + ": " + nccl().GetErrorString(r);
    return cudaErrorUnknown;
  }
  cudaError_t exchange(const std::vector<char *> &p, size_t pb, const std::vector<int> &lo, const std::vector<int> &hi,
                       int g, cudaStream_t st) override {
    const int esz = dtype == ncclFloat64 ? 8 : 4;
    const size_t cnt = g * pb / esz;
    char *a = p[0];
    if (!comm) return check(3 /* ncclInternalError */, "halo exchange on an aborted communicator");
    ncclResult_t r = nccl().GroupStart();
    if (q > 0) {
      if (!r) r = nccl().Send(a + (int64_t)lo[0] * pb, cnt, dtype, q - 1, comm, st);
      if (!r) r = nccl().Recv(a + (int64_t)(lo[0] - g) * pb, cnt, dtype, q - 1, comm, st);
    }
    if (q + 1 < P) {
      if (!r) r = nccl().Send(a + (int64_t)(hi[0] - g) * pb, cnt, dtype, q + 1, comm, st);
      if (!r) r = nccl().Recv(a + (int64_t)hi[0] * pb, cnt, dtype, q + 1, comm, st);
    }
    ncclResult_t r2 = nccl().GroupEnd();
    return check(r ? r : r2, "halo exchange");
  }
  cudaError_t allgather(char *full, size_t pb, int lo, int rows, int esz, cudaStream_t st) override {
    const size_t cnt = rows * pb / esz;
    return check(nccl().AllGather(full + (int64_t)lo * pb, full + (int64_t)(lo - q * rows) * pb, cnt, dtype, comm, st),
                 "agglomeration all-gather");
  }
  cudaError_t allreduce_max_u64(unsigned long long *d, int n, cudaStream_t st) override {
    return check(nccl().AllReduce(d, d, n, ncclUint64, ncclMax, comm, st), "norm all-reduce");
  }
  cudaError_t allreduce_sum_f64(double *d, int n, cudaStream_t st) override {
    return check(nccl().AllReduce(d, d, n, ncclFloat64, ncclSum, comm, st), "norm all-reduce");
  }
  std::string error() const override { return err; }
  std::string poll() override {
    if (!comm || !nccl().CommGetAsyncError) return comm ? "" : err;
    ncclResult_t a = 0;
    ncclResult_t r = nccl().CommGetAsyncError(comm, &a);
    if (r == 0 && (a == 0 || a == 7 /* ncclInProgress */)) return "";
    err = std::string("NCCL asynchronous error: ") + nccl().GetErrorString(r ? r : a);
    if (nccl().CommAbort) nccl().CommAbort(comm);
    else nccl().CommDestroy(comm);
    comm = nullptr;
    return err;
  }
};


Comm2 *make_loop_comm(int P) {
  auto *c = new LoopComm();
  c->P = P;
  return c;
}

Comm2 *make_nccl_comm(int P, int rank, const void *id, int esz, std::string *err) {
  auto *nc = new NcclComm();
  if (!nc->init(P, rank, id, esz)) {
    *err = nc->err;
    delete nc;
    return nullptr;
  }
  return nc;
}

int nccl_unique_id(void *out, std::string *err) {
  if (!nccl().load()) {
    *err = nccl().why;
    return MG_ENCCL;
  }
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != 0) {
    *err = "ncclGetUniqueId failed";
    return MG_ENCCL;
  }
  std::memcpy(out, &id, sizeof id);
  return MG_OK;
}

}  // namespace mg
