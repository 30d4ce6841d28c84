// Native multi-GPU data plane: an NCCL communicator over the
// ranks of a cell partition. The interface exchange of a rank-spanning sync
// is neighbour-only — grouped ncclSend / ncclRecv with each peer rank that
// shares a macro face, edge or vertex, carrying exactly the replica values
// the peer's member-order sums read (XPlan::sends / recvs, bt_xchg.cu) — and
// dot partials go through ncclAllReduce. Everything is enqueued on the
// caller's stream, so an apply, a smoother sweep or a whole V-cycle stays
// stream-ordered (and capturable) with no host round trip and no Python.
//
// NCCL is resolved at bt_comm_create with dlopen("libnccl.so.2"): inside a
// process that already loaded NCCL (e.g. through torch) that is the same
// library, so the library has no link-time NCCL dependency. Types and enum
// values come from nccl.h (stable across NCCL 2.x).
#include <dlfcn.h>
#include <cmath>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bt_internal.hpp"

struct bt_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

namespace bt {
namespace {
struct Nccl {
  void* lib = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      err = std::string("bt_comm: cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("bt_comm: libnccl lacks ") + name;
      return p;
    };
    n.get_unique_id = (decltype(n.get_unique_id))sym("ncclGetUniqueId");
    n.init_rank = (decltype(n.init_rank))sym("ncclCommInitRank");
    n.destroy = (decltype(n.destroy))sym("ncclCommDestroy");
    n.send = (decltype(n.send))sym("ncclSend");
    n.recv = (decltype(n.recv))sym("ncclRecv");
    n.group_start = (decltype(n.group_start))sym("ncclGroupStart");
    n.group_end = (decltype(n.group_end))sym("ncclGroupEnd");
    n.all_reduce = (decltype(n.all_reduce))sym("ncclAllReduce");
    n.error_string = (decltype(n.error_string))sym("ncclGetErrorString");
    if (err.empty()) n.lib = h;
  });
  if (!n.lib) raise(BT_RUNTIME_ERROR, err);
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    raise(BT_RUNTIME_ERROR, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}
}  // namespace

void comm_check(const bt_comm* c, int rank, int nranks) {
  if (!c || !c->comm) raise(BT_LOGIC_ERROR, "bt_comm: communicator destroyed or never created");
  if (c->rank != rank || c->nranks != nranks)
    raise(BT_LOGIC_ERROR, "bt_comm: the communicator's (rank, nranks) is not the grid's partition");
}

void comm_sendrecv(bt_comm* c, const std::vector<int>& peers, const std::vector<int64_t>& send_off,
                   const std::vector<int64_t>& recv_off, const double* sendbuf, double* recvbuf, cudaStream_t s) {
  const Nccl& n = nccl();
  check(n.group_start(), "ncclGroupStart");
  for (size_t i = 0; i < peers.size(); ++i) {
    const size_t ns = (size_t)(send_off[i + 1] - send_off[i]), nr = (size_t)(recv_off[i + 1] - recv_off[i]);
    if (ns) check(n.send(sendbuf + send_off[i], ns, ncclFloat64, peers[i], c->comm, s), "ncclSend");
    if (nr) check(n.recv(recvbuf + recv_off[i], nr, ncclFloat64, peers[i], c->comm, s), "ncclRecv");
  }
  check(n.group_end(), "ncclGroupEnd");
}

void comm_allreduce(bt_comm* c, double* buf, int64_t cnt, cudaStream_t s) {
  if (cnt <= 0) return;
  // every element has one nonzero contribution (the owning rank's), so the
  // sum is exact in any reduction order
  check(nccl().all_reduce(buf, buf, (size_t)cnt, ncclFloat64, ncclSum, c->comm, s), "ncclAllReduce");
}

}  // namespace bt

using namespace bt;

extern "C" {

bt_status bt_comm_unique_id(uint8_t id[128]) {
  BT_TRY
  if (!id) raise(BT_INVALID_ARGUMENT, "bt_comm_unique_id: id required");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof u);
  BT_CATCH
}

bt_status bt_comm_create(const uint8_t id[128], int rank, int nranks, int device, bt_comm** out) {
  BT_TRY
  if (!id || !out) raise(BT_INVALID_ARGUMENT, "bt_comm_create: id and out required");
  if (nranks < 1 || rank < 0 || rank >= nranks) raise(BT_INVALID_ARGUMENT, "bt_comm_create: bad rank / nranks");
  *out = nullptr;
  BT_CUDA(cudaSetDevice(device));
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  auto c = std::make_unique<bt_comm>();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  check(nccl().init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
  *out = c.release();
  BT_CATCH
}

void bt_comm_destroy(bt_comm* c) {
  if (!c) return;
  if (c->comm) {
    cudaSetDevice(c->device);
    try {
      nccl().destroy(c->comm);
    } catch (...) {
    }
  }
  delete c;
}

}  // extern "C"
