// Multi-GPU exchange of the monolithic scheme: macro points
// are sharded in contiguous equal blocks over the ranks of one box, one engine
// handle per device, and after every increment / macro iteration each rank
// needs every point's condensed response. The per-point records
// {Σ (nc) | C (nt) | ‖r‖ | status} are packed on the device straight into
// this rank's block of the receive buffer and all-gathered in place over NCCL
// (NVLink / NVSwitch); a max all-reduce of the local "some point failed" flag
// gives the lockstep termination test. This is the only collective on the
// path: assembly, factorisation and condensation never communicate.
//
// libnccl.so.2 is dlopen'ed at first use (the process's NCCL — torch's bundled
// one when torch is loaded — or the system one), so the engine library has no
// link-time NCCL dependency. Reference: the points are independent
// ("parallelize over macro integration points"); the
// records are what fe2.macro_step consumes.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <type_traits>

#include "common.hpp"
#include "host_util.cuh"

namespace fe2 {

namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclCommUserRank) comm_user_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string err;

  static const Nccl& get() {
    static const Nccl s = load();
    check(s.err.empty(), Code::rank, s.err);
    return s;
  }

 private:
  static Nccl load() {
    Nccl s;
    void* lib = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!lib) {
      s.err = "cannot load NCCL (libnccl.so.2)";
      return s;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (!fn && s.err.empty()) s.err = std::string("NCCL symbol missing: ") + name;
    };
    sym(s.get_unique_id, "ncclGetUniqueId");
    sym(s.comm_init_rank, "ncclCommInitRank");
    sym(s.comm_destroy, "ncclCommDestroy");
    sym(s.comm_count, "ncclCommCount");
    sym(s.comm_user_rank, "ncclCommUserRank");
    sym(s.all_gather, "ncclAllGather");
    sym(s.all_reduce, "ncclAllReduce");
    sym(s.error_string, "ncclGetErrorString");
    return s;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Failure(Code::rank, std::string("NCCL ") + what + " failed: " + Nccl::get().error_string(r));
}

// One thread per (point, record field): record p = [sigma(nc) | C(nt) | res | status]
// at out[p * R]; flag |= (status != 0).
__global__ void k_pack_records(int64_t P, int nc, int nt, const double* __restrict__ sigma,
                               const double* __restrict__ C, const double* __restrict__ res,
                               const int* __restrict__ status, double* __restrict__ out, int* __restrict__ flag) {
  const int R = nc + nt + 2;
  const int64_t total = P * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = e / R;
    const int f = static_cast<int>(e - p * R);
    double v;
    if (f < nc) {
      v = sigma[p * nc + f];
    } else if (f < nc + nt) {
      v = C[p * nt + (f - nc)];
    } else if (f == nc + nt) {
      v = res[p];
    } else {
      const int s = status[p];
      v = static_cast<double>(s);
      if (s != 0) atomicOr(flag, 1);
    }
    out[e] = v;
  }
}

}  // namespace

// Pack this rank's records into d_all[rank block], all-gather in place, and
// max-reduce the failure flag (host result; synchronises `stream`).
void exchange_records(int device, cudaStream_t stream, void* comm_v, int64_t P, int nc, int nt, const double* d_sigma,
                      const double* d_C, const double* d_res, const int* d_status, double* d_all, int* any_failed) {
  const Nccl& N = Nccl::get();
  auto comm = static_cast<ncclComm_t>(comm_v);
  check(comm != nullptr, Code::config, "null NCCL communicator");
  check(d_sigma && d_C && d_res && d_status && d_all, Code::config, "null device buffer");
  int world = 0, rank = 0;
  nccl_check(N.comm_count(comm, &world), "ncclCommCount");
  nccl_check(N.comm_user_rank(comm, &rank), "ncclCommUserRank");
  CK(cudaSetDevice(device));
  const int R = nc + nt + 2;
  const size_t count = static_cast<size_t>(P) * R;
  double* mine = d_all + static_cast<size_t>(rank) * count;
  int* flag = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), stream));
  CK(cudaMemsetAsync(flag, 0, sizeof(int), stream));
  if (P > 0) {
    const int64_t blocks = (static_cast<int64_t>(count) + 255) / 256;
    k_pack_records<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, stream>>>(
        P, nc, nt, d_sigma, d_C, d_res, d_status, mine, flag);
    CK(cudaGetLastError());
  }
  // in place: sendbuff = recvbuff + rank * sendcount
  nccl_check(N.all_gather(mine, d_all, count, ncclFloat64, comm, stream), "ncclAllGather");
  nccl_check(N.all_reduce(flag, flag, 1, ncclInt32, ncclMax, comm, stream), "ncclAllReduce");
  int h = 0;
  CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CK(cudaFreeAsync(flag, stream));
  CK(cudaStreamSynchronize(stream));
  if (any_failed) *any_failed = h;
}

}  // namespace fe2

using namespace fe2;

extern "C" {

int fe2_nccl_get_unique_id(void* id128) {
  return guard([&] {
    check(id128 != nullptr, Code::config, "null id buffer");
    ncclUniqueId id;
    nccl_check(Nccl::get().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof(id));
  });
}

int fe2_nccl_comm_init(int device, int nranks, int rank, const void* id128, void** comm) {
  return guard([&] {
    check(id128 != nullptr && comm != nullptr, Code::config, "bad arguments");
    check(nranks >= 1 && rank >= 0 && rank < nranks, Code::config, "rank out of range");
    require_device(device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    nccl_check(Nccl::get().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int fe2_nccl_comm_destroy(void* comm) {
  return guard([&] {
    if (comm) nccl_check(Nccl::get().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

}  // extern "C"
