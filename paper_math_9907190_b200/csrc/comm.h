// comm.h -- halo / gather / reduce transports of the multi-GPU slab solvers
// (dist2.cu: 2D y-slabs, dist3.cu: 3D z-slabs).  A slab array family is
// given per local rank as a virtual global-row-0 pointer with a row pitch in
// bytes ("row" = a 2D row or a 3D plane); rows [lo, hi) are owned.
#pragma once
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/mg.h"

namespace mg {

struct Comm2 {
  int P = 1;
  virtual ~Comm2() {}
  // ghost rows [lo-g, lo) and [hi, hi+g) of every local rank from its neighbours
  virtual cudaError_t exchange(const std::vector<char *> &p, size_t pitch_b, const std::vector<int> &lo,
                               const std::vector<int> &hi, int g, cudaStream_t st) = 0;
  // full array (virtual row 0 pointer): own rows [lo, lo+rows) -> every rank
  virtual cudaError_t allgather(char *full, size_t pitch_b, int lo, int rows, int esz, cudaStream_t st) = 0;
  virtual cudaError_t allreduce_max_u64(unsigned long long *d, int n, cudaStream_t st) = 0;
  virtual cudaError_t allreduce_sum_f64(double *d, int n, cudaStream_t st) = 0;
  virtual std::string error() const { return ""; }
  // asynchronous transport failure (NCCL: ncclCommGetAsyncError); on error the
  // communicator is aborted and the message returned ("" = healthy)
  virtual std::string poll() { return ""; }
};

// Sticky status of a slab solver's enqueue_* calls: the first failed step
// (kernel launch, halo exchange, all-gather, all-reduce) is kept until the
// ABI takes it (ImplBase::take_status), then the graph being captured is
// dropped and the call fails with MG_ENCCL / MG_ECUDA.
struct TransportStatus {
  int code = MG_OK;
  std::string msg;
  void note(cudaError_t e, const Comm2 *c, const char *what) {
    if (e == cudaSuccess || code != MG_OK) return;
    const std::string ce = c ? c->error() : std::string();
    code = ce.empty() ? MG_ECUDA : MG_ENCCL;
    msg = std::string(what) + ": " + (ce.empty() ? cudaGetErrorString(e) : ce);
  }
  int take(std::string *m, Comm2 *c) {
    if (code == MG_OK && c) {
      const std::string a = c->poll();
      if (!a.empty()) {
        code = MG_ENCCL;
        msg = a;
      }
    }
    const int r = code;
    if (m) *m = msg;
    code = MG_OK;
    msg.clear();
    return r;
  }
};

// P virtual ranks in one process on one GPU: device-to-device copies.
Comm2 *make_loop_comm(int P);
// One process per GPU over NCCL (libnccl.so.2 loaded at run time); nullptr
// and *err on failure.  esz = element size of the arrays exchanged.
Comm2 *make_nccl_comm(int P, int rank, const void *nccl_id, int esz, std::string *err);
int nccl_unique_id(void *out, std::string *err);

}  // namespace mg
