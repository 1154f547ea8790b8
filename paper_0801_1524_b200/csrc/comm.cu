// comm.cu -- NCCL inside the library (SURVEY.md §8(b) multi-GPU contract,
// §8(e) exchange): the level-m charge exchange of a sharded plan as grouped
// ncclSend/ncclRecv on the plan stream, and the all-gather of u.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): if the process
// already has an NCCL loaded (torch.distributed's), that instance is used, so
// libsft never brings a second NCCL into a process.  Only nccl.h's types are
// used at compile time.
//
// Communicators are cached per (ncclUniqueId, rank, world, device): the first
// sft_plan of a rank with a given id calls ncclCommInitRank (a collective: all
// ranks must plan concurrently), later plans with the same id reuse it, so a
// plan/apply/destroy loop pays for the init once.  sft_nccl_release(id)
// destroys it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "sft_internal.cuh"

namespace sft {

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
};

std::mutex g_mu;

const NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  std::lock_guard<std::mutex> lk(g_mu);
  if (tried) return a;
  tried = true;
  // an NCCL already in the process first (torch's), else the loader's search path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    a.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    return a;
  }
  bool all = true;
  auto sym = [&](auto& fp, const char* name) {
    fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
    if (!fp) {
      all = false;
      a.err = std::string("libnccl.so.2 lacks ") + name;
    }
  };
  sym(a.GetUniqueId, "ncclGetUniqueId");
  sym(a.CommInitRank, "ncclCommInitRank");
  sym(a.CommDestroy, "ncclCommDestroy");
  sym(a.GetErrorString, "ncclGetErrorString");
  sym(a.Send, "ncclSend");
  sym(a.Recv, "ncclRecv");
  sym(a.AllGather, "ncclAllGather");
  sym(a.GroupStart, "ncclGroupStart");
  sym(a.GroupEnd, "ncclGroupEnd");
  a.ok = all;
  return a;
}

using CommKey = std::tuple<std::string, int, int, int>;  // id bytes, rank, world, device
std::map<CommKey, ncclComm_t>& comm_cache() {
  static std::map<CommKey, ncclComm_t> m;
  return m;
}

std::string nccl_msg(const NcclApi& a, ncclResult_t r, const char* what) {
  return std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error");
}

}  // namespace

int nccl_comm_get(const void* id128, int rank, int world, void** out, std::string* err) {
  const NcclApi& a = api();
  if (!a.ok) {
    *err = a.err;
    return SFT_E_NCCL;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    *err = "cudaGetDevice failed";
    return SFT_E_CUDA;
  }
  const CommKey key(std::string(static_cast<const char*>(id128), NCCL_UNIQUE_ID_BYTES), rank, world, dev);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = comm_cache().find(key);
    if (it != comm_cache().end()) {
      *out = it->second;
      return SFT_OK;
    }
  }
  // (outside the lock: ncclCommInitRank blocks until every rank has joined)
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = a.CommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) {
    *err = nccl_msg(a, r, "ncclCommInitRank");
    return SFT_E_NCCL;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  comm_cache()[key] = c;
  *out = c;
  return SFT_OK;
}

// Level-m exchange: segment q of `send` (send_counts[q] complex128 in rank
// order) goes to rank q; rank q's segment for us lands at its offset in `recv`
// (the peers' segments concatenated in rank order).  One NCCL group, so every
// pair's transfer runs concurrently; stream-ordered on s.
int nccl_exchange(void* comm, const double2* send, const int64_t* send_counts, double2* recv,
                  const int64_t* recv_counts, int world, cudaStream_t s, std::string* err) {
  const NcclApi& a = api();
  if (!a.ok) {
    *err = a.err;
    return SFT_E_NCCL;
  }
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = a.GroupStart();
  int64_t so = 0, ro = 0;
  for (int q = 0; q < world && r == ncclSuccess; ++q) {
    if (send_counts[q] > 0) r = a.Send(send + so, 2 * (size_t)send_counts[q], ncclFloat64, q, c, s);
    if (r == ncclSuccess && recv_counts[q] > 0) r = a.Recv(recv + ro, 2 * (size_t)recv_counts[q], ncclFloat64, q, c, s);
    so += send_counts[q];
    ro += recv_counts[q];
  }
  ncclResult_t r2 = a.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    *err = nccl_msg(a, r, "level-m exchange (ncclSend/ncclRecv)");
    return SFT_E_NCCL;
  }
  return SFT_OK;
}

// u all-gather: every rank contributes `count` complex128 (its targets in
// sorted order, padded to the largest rank's count); recv = [world][count].
int nccl_allgather(void* comm, const double2* send, double2* recv, int64_t count, cudaStream_t s, std::string* err) {
  const NcclApi& a = api();
  if (!a.ok) {
    *err = a.err;
    return SFT_E_NCCL;
  }
  ncclResult_t r = a.AllGather(send, recv, 2 * (size_t)count, ncclFloat64, static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) {
    *err = nccl_msg(a, r, "u all-gather (ncclAllGather)");
    return SFT_E_NCCL;
  }
  return SFT_OK;
}

}  // namespace sft

extern "C" int sft_nccl_unique_id(void* id128) {
  if (!id128) return SFT_E_ARG;
  const sft::NcclApi& a = sft::api();
  if (!a.ok) return SFT_E_NCCL;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return SFT_E_NCCL;
  std::memcpy(id128, &id, sizeof(id));
  return SFT_OK;
}

extern "C" int sft_nccl_release(const void* id128) {
  if (!id128) return SFT_E_ARG;
  const sft::NcclApi& a = sft::api();
  if (!a.ok) return SFT_OK;  // nothing can have been created
  const std::string idb(static_cast<const char*>(id128), NCCL_UNIQUE_ID_BYTES);
  std::lock_guard<std::mutex> lk(sft::g_mu);
  auto& m = sft::comm_cache();
  for (auto it = m.begin(); it != m.end();) {
    if (std::get<0>(it->first) == idb) {
      a.CommDestroy(it->second);
      it = m.erase(it);
    } else {
      ++it;
    }
  }
  return SFT_OK;
}
