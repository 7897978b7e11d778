// Multi-GPU exchange of the monolithic scheme: macro points
// are sharded in contiguous blocks over the ranks of one box (any sizes: blocks are
// padded to the largest rank's count in the gathered buffer), one engine
// handle per device, and after every increment / macro iteration each rank
// needs every point's condensed response. The per-point records
// {Σ (nc) | C (nt) | ‖r‖ | status} are packed on the device straight into
// this rank's block of the receive buffer and all-gathered in place over NCCL
// (NVLink / NVSwitch); a max all-reduce of the local "some point failed" and "some
// point above the residual tolerance" flags gives the lockstep termination test. This is the only collective on the
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

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>
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

// One thread per (row, record field) of this rank's padded block of P_max rows:
// record p = [sigma(nc) | C(nt) | res | status] at out[p * R]; rows p >= P are padding
// (NaN, status -1). flags[0] |= (status > 0): a failed point; flags[1] |= (res > res_tol):
// a point not yet converged (the monolithic iteration's lockstep termination test).
__global__ void k_pack_records(int64_t P, int64_t P_max, int nc, int nt, const double* __restrict__ sigma,
                               const double* __restrict__ C, const double* __restrict__ res,
                               const int* __restrict__ status, double res_tol, double* __restrict__ out,
                               int* __restrict__ flags) {
  const int R = nc + nt + 2;
  const int64_t total = P_max * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = e / R;
    const int f = static_cast<int>(e - p * R);
    double v;
    if (p >= P) {
      v = f == nc + nt + 1 ? -1.0 : __longlong_as_double(0x7ff8000000000000LL);
    } else if (f < nc) {
      v = sigma[p * nc + f];
    } else if (f < nc + nt) {
      v = C[p * nt + (f - nc)];
    } else if (f == nc + nt) {
      v = res[p];
      if (!(v <= res_tol)) atomicOr(flags + 1, 1);
    } else {
      const int s = status[p];
      v = static_cast<double>(s);
      if (s > 0) atomicOr(flags, 1);
    }
    out[e] = v;
  }
}

}  // namespace

// Block layout of the exchange: every rank's P_local (one in-place ncclAllGather of an
// int64 per rank; host-synchronising, done once per communicator by the caller).
void exchange_layout(int device, cudaStream_t stream, void* comm_v, int64_t P, int64_t* scratch,
                     ExchangeLayout* out) {
  const Nccl& N = Nccl::get();
  auto comm = static_cast<ncclComm_t>(comm_v);
  check(comm != nullptr, Code::config, "null NCCL communicator");
  int world = 0, rank = 0;
  nccl_check(N.comm_count(comm, &world), "ncclCommCount");
  nccl_check(N.comm_user_rank(comm, &rank), "ncclCommUserRank");
  check(world <= kMaxRanks, Code::rank, "too many ranks for the exchange layout");
  CK(cudaSetDevice(device));
  int64_t* d = scratch;  // kMaxRanks int64 of device scratch owned by the handle
  CK(cudaMemcpyAsync(d + rank, &P, sizeof(int64_t), cudaMemcpyHostToDevice, stream));
  nccl_check(N.all_gather(d + rank, d, 1, ncclInt64, comm, stream), "ncclAllGather(P_local)");
  std::vector<int64_t> counts(world);
  CK(cudaMemcpyAsync(counts.data(), d, world * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  out->comm = comm_v;
  out->world = world;
  out->rank = rank;
  out->P_local = P;
  out->P_max = 0;
  out->P_total = 0;
  for (int r = 0; r < world; ++r) {
    check(counts[r] >= 0, Code::rank, "bad point count from a rank");
    out->P_max = std::max(out->P_max, counts[r]);
    out->P_total += counts[r];
    out->counts[r] = counts[r];
  }
}

// Pack this rank's records into d_all[rank * P_max * R ...] (padding rows beyond P_local),
// all-gather in place, max-reduce the two flags; with flags_host the flags are copied
// (pinned h_flags) and the stream synchronised, otherwise everything stays asynchronous.
void exchange_records(int device, cudaStream_t stream, const ExchangeLayout& L, int nc, int nt,
                      const double* d_sigma, const double* d_C, const double* d_res, const int* d_status,
                      double res_tol, double* d_all, int* d_flags, int* h_flags, int* flags_host) {
  const Nccl& N = Nccl::get();
  auto comm = static_cast<ncclComm_t>(L.comm);
  check(d_sigma && d_C && d_res && d_status && d_all, Code::config, "null device buffer");
  CK(cudaSetDevice(device));
  const int R = nc + nt + 2;
  const size_t count = static_cast<size_t>(L.P_max) * R;
  double* mine = d_all + static_cast<size_t>(L.rank) * count;
  CK(cudaMemsetAsync(d_flags, 0, 2 * sizeof(int), stream));
  if (count > 0) {
    const int64_t blocks = (static_cast<int64_t>(count) + 255) / 256;
    k_pack_records<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, stream>>>(
        L.P_local, L.P_max, nc, nt, d_sigma, d_C, d_res, d_status, res_tol, mine, d_flags);
    CK(cudaGetLastError());
  }
  // in place: sendbuff = recvbuff + rank * sendcount
  nccl_check(N.all_gather(mine, d_all, count, ncclFloat64, comm, stream), "ncclAllGather");
  nccl_check(N.all_reduce(d_flags, d_flags, 2, ncclInt32, ncclMax, comm, stream), "ncclAllReduce");
  if (flags_host) {
    CK(cudaMemcpyAsync(h_flags, d_flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    flags_host[0] = h_flags[0];
    flags_host[1] = h_flags[1];
  }
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
