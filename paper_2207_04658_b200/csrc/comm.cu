// comm.cu -- NCCL point-to-point for the slab decomposition: grouped
// ncclSend / ncclRecv with the two z-neighbours on the ctx stream.  NCCL is resolved
// with dlopen so the library loads on machines without it; the communicator is
// built from a unique id the caller broadcasts (e.g. with torch.distributed).
#include <dlfcn.h>

#include <mutex>
#include <string>

#include <nccl.h>

#include "comm.h"

namespace qmpm {

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  bool ok = false;
};

std::mutex g_mu;
NcclApi g_api;

template <class T>
bool sym(void* h, const char* name, T& fn) {
  fn = reinterpret_cast<T>(dlsym(h, name));
  return fn != nullptr;
}

bool load(std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_api.ok) return true;
  void* h = nullptr;
  for (const char* c : {"libnccl.so.2", "libnccl.so", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"})
    if ((h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    err = "libnccl.so.2 not found";
    return false;
  }
  g_api.ok = sym(h, "ncclGetUniqueId", g_api.getUniqueId) && sym(h, "ncclCommInitRank", g_api.commInitRank) &&
             sym(h, "ncclCommDestroy", g_api.commDestroy) && sym(h, "ncclSend", g_api.send) &&
             sym(h, "ncclRecv", g_api.recv) && sym(h, "ncclGroupStart", g_api.groupStart) &&
             sym(h, "ncclGroupEnd", g_api.groupEnd) && sym(h, "ncclGetErrorString", g_api.errstr) &&
             sym(h, "ncclAllReduce", g_api.allReduce);
  if (!g_api.ok) err = "incomplete libnccl";
  return g_api.ok;
}

}  // namespace

struct NcclComm {
  ncclComm_t comm;
  int nranks, rank;
};

bool nccl_unique_id(unsigned char id[128], std::string& err) {
  if (!load(err)) return false;
  ncclUniqueId u;
  ncclResult_t r = g_api.getUniqueId(&u);
  if (r != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + g_api.errstr(r);
    return false;
  }
  static_assert(sizeof(u.internal) == 128, "NCCL unique id is 128 bytes");
  for (int i = 0; i < 128; ++i) id[i] = (unsigned char)u.internal[i];
  return true;
}

NcclComm* nccl_connect(const unsigned char id[128], int nranks, int rank, std::string& err) {
  if (!load(err)) return nullptr;
  ncclUniqueId u;
  for (int i = 0; i < 128; ++i) u.internal[i] = (char)id[i];
  NcclComm* c = new NcclComm{nullptr, nranks, rank};
  ncclResult_t r = g_api.commInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + g_api.errstr(r);
    delete c;
    return nullptr;
  }
  return c;
}

void nccl_destroy(NcclComm* c) {
  if (!c) return;
  if (g_api.ok && c->comm) g_api.commDestroy(c->comm);
  delete c;
}

bool nccl_exchange(NcclComm* c, const P2P& x, cudaStream_t st, std::string& err) {
  ncclResult_t r = g_api.groupStart();
  const int dn = c->rank - 1, up = c->rank + 1;
  if (r == ncclSuccess && dn >= 0 && x.send_dn_bytes)
    r = g_api.send(x.send_dn, x.send_dn_bytes, ncclUint8, dn, c->comm, st);
  if (r == ncclSuccess && up < c->nranks && x.send_up_bytes)
    r = g_api.send(x.send_up, x.send_up_bytes, ncclUint8, up, c->comm, st);
  if (r == ncclSuccess && dn >= 0 && x.recv_dn_bytes)
    r = g_api.recv(x.recv_dn, x.recv_dn_bytes, ncclUint8, dn, c->comm, st);
  if (r == ncclSuccess && up < c->nranks && x.recv_up_bytes)
    r = g_api.recv(x.recv_up, x.recv_up_bytes, ncclUint8, up, c->comm, st);
  ncclResult_t r2 = g_api.groupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    err = std::string("NCCL exchange: ") + g_api.errstr(r);
    return false;
  }
  return true;
}

bool nccl_allreduce_max_u32(NcclComm* c, unsigned int* v, cudaStream_t st, std::string& err) {
  ncclResult_t r = g_api.allReduce(v, v, 1, ncclUint32, ncclMax, c->comm, st);
  if (r != ncclSuccess) {
    err = std::string("NCCL all-reduce: ") + g_api.errstr(r);
    return false;
  }
  return true;
}

}  // namespace qmpm
