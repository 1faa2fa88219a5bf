// comm.cu — NCCL and in-process transports of the Comm interface (comm.cuh).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <list>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"

// In-process group: W ranks (contexts) of one process, one host thread each.
struct mpr_group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  struct Post {
    const void* ptr = nullptr;
    size_t count = 0;
  };
  std::vector<Post> post;
  // point-to-point mailbox: the k-th message from src to dst matches dst's k-th receive
  // from src (NCCL's ordering rule); the sender waits until the receiver has copied it
  struct Msg {
    int src, dst;
    uint64_t seq;
    const void* ptr;
    size_t bytes;
    bool done;
  };
  std::list<Msg> msgs;
  std::vector<uint64_t> send_seq, recv_seq;  // [src * world + dst]
};

namespace mpr {

size_t comm_type_size(CommType t) {
  switch (t) {
    case CT_U8: return 1;
    case CT_I32: return 4;
    case CT_F32: return 4;
    case CT_I64: return 8;
    case CT_U64: return 8;
    case CT_F64: return 8;
  }
  return 1;
}

namespace {

// ------------------------------------------------------------------ NCCL, dlopen'd
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommCuDevice)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// The process's libnccl.so.2: the copy already loaded (e.g. torch's) if there is one, so a
// communicator made by the caller and the calls made here go to the same library.
NcclApi load_nccl() {
  NcclApi a;
  const char* env = std::getenv("MPR_NCCL_LIB");
  void* h = nullptr;
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.why = std::string("libnccl.so.2 not found: ") + dlerror();
    return a;
  }
#define SYM(field, name)                                                    \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));            \
  if (!a.field) {                                                           \
    a.why = std::string("libnccl: missing symbol ") + name;                 \
    return a;                                                               \
  }
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(CommCount, "ncclCommCount");
  SYM(CommUserRank, "ncclCommUserRank");
  SYM(CommCuDevice, "ncclCommCuDevice");
  SYM(AllReduce, "ncclAllReduce");
  SYM(Broadcast, "ncclBroadcast");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  a.ok = true;
  return a;
}

NcclApi& nccl() {
  static NcclApi api = load_nccl();
  return api;
}

ncclDataType_t nccl_type(CommType t) {
  switch (t) {
    case CT_U8: return ncclUint8;
    case CT_I32: return ncclInt32;
    case CT_I64: return ncclInt64;
    case CT_U64: return ncclUint64;
    case CT_F32: return ncclFloat32;
    case CT_F64: return ncclFloat64;
  }
  return ncclUint8;
}

ncclRedOp_t nccl_op(CommOp op) { return op == OP_MIN ? ncclMin : op == OP_MAX ? ncclMax : ncclSum; }

class NcclComm final : public Comm {
 public:
  ncclComm_t comm = nullptr;
  bool stream_ordered() const override { return true; }
  const char* name() const override { return "nccl"; }

  mpr_status check(ncclResult_t r, const char* where) {
    if (r == ncclSuccess) return MPR_OK;
    err = std::string(where) + ": " + nccl().GetErrorString(r);
    return MPR_ERR_NCCL;
  }

  mpr_status allreduce(void* buf, size_t count, CommType t, CommOp op, cudaStream_t st) override {
    if (count == 0) return MPR_OK;
    return check(nccl().AllReduce(buf, buf, count, nccl_type(t), nccl_op(op), comm, st), "ncclAllReduce");
  }

  mpr_status exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, CommType t,
                      cudaStream_t st) override {
    if (sends.empty() && recvs.empty()) return MPR_OK;
    mpr_status s = check(nccl().GroupStart(), "ncclGroupStart");
    if (s != MPR_OK) return s;
    mpr_status first = MPR_OK;
    for (const P2P& p : sends)
      if (p.count && first == MPR_OK) first = check(nccl().Send(p.ptr, p.count, nccl_type(t), p.peer, comm, st), "ncclSend");
    for (const P2P& p : recvs)
      if (p.count && first == MPR_OK) first = check(nccl().Recv(p.ptr, p.count, nccl_type(t), p.peer, comm, st), "ncclRecv");
    s = check(nccl().GroupEnd(), "ncclGroupEnd");
    return first != MPR_OK ? first : s;
  }

  mpr_status allgatherv(const void* send, void* recv, const std::vector<size_t>& counts,
                        const std::vector<size_t>& displs, CommType t, cudaStream_t st) override {
    const size_t es = comm_type_size(t);
    char* r = static_cast<char*>(recv);
    char* mine = r + displs[rank] * es;
    if (send != mine && counts[rank]) {
      cudaError_t e = cudaMemcpyAsync(mine, send, counts[rank] * es, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) {
        err = std::string("allgatherv copy: ") + cudaGetErrorString(e);
        return MPR_ERR_CUDA;
      }
    }
    // variable counts: one broadcast per root, grouped
    mpr_status s = check(nccl().GroupStart(), "ncclGroupStart");
    if (s != MPR_OK) return s;
    mpr_status first = MPR_OK;
    for (int w = 0; w < world; ++w) {
      char* p = r + displs[w] * es;
      if (counts[w] && first == MPR_OK) first = check(nccl().Broadcast(p, p, counts[w], nccl_type(t), w, comm, st), "ncclBroadcast");
    }
    s = check(nccl().GroupEnd(), "ncclGroupEnd");
    return first != MPR_OK ? first : s;
  }

  mpr_status broadcast(void* buf, size_t count, CommType t, int root, cudaStream_t st) override {
    if (count == 0) return MPR_OK;
    return check(nccl().Broadcast(buf, buf, count, nccl_type(t), root, comm, st), "ncclBroadcast");
  }
};

// ------------------------------------------------------------- in-process group
class GroupComm final : public Comm {
 public:
  mpr_group* g = nullptr;
  bool stream_ordered() const override { return false; }
  const char* name() const override { return "group"; }

  // Generation barrier of the group's host threads (timeout: MPR_GROUP_TIMEOUT_S, 600 s).
  mpr_status barrier() {
    static const int timeout_s = [] {
      const char* v = std::getenv("MPR_GROUP_TIMEOUT_S");
      return v ? std::atoi(v) : 600;
    }();
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->aborted) {
      err = "group aborted by another rank";
      return MPR_ERR_STATE;
    }
    const uint64_t my = g->gen;
    if (++g->arrived == g->world) {
      g->arrived = 0;
      ++g->gen;
      g->cv.notify_all();
      return MPR_OK;
    }
    if (!g->cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return g->gen != my || g->aborted; })) {
      g->aborted = true;
      g->cv.notify_all();
      err = "group barrier timed out (a rank did not reach the collective)";
      return MPR_ERR_STATE;
    }
    if (g->aborted && g->gen == my) {
      err = "group aborted by another rank";
      return MPR_ERR_STATE;
    }
    return MPR_OK;
  }

  mpr_status cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return MPR_OK;
    err = std::string(where) + ": " + cudaGetErrorString(e);
    return MPR_ERR_CUDA;
  }

  // post this rank's buffer, wait until every rank has posted (its data complete)
  mpr_status publish(const void* ptr, size_t count, cudaStream_t st) {
    mpr_status s = cuda(cudaStreamSynchronize(st), "group: stream sync");
    if (s != MPR_OK) return s;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->post[rank].ptr = ptr;
      g->post[rank].count = count;
    }
    return barrier();
  }

  // wait on the group's condition variable for pred(), with the barrier's timeout
  template <class Pred>
  mpr_status wait_for(std::unique_lock<std::mutex>& lk, Pred pred, const char* what) {
    const char* v = std::getenv("MPR_GROUP_TIMEOUT_S");
    const int timeout_s = v ? std::atoi(v) : 600;
    if (!g->cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return pred() || g->aborted; })) {
      g->aborted = true;
      g->cv.notify_all();
      err = std::string("group: timed out waiting for ") + what;
      return MPR_ERR_STATE;
    }
    if (!pred()) {
      err = "group aborted by another rank";
      return MPR_ERR_STATE;
    }
    return MPR_OK;
  }

  // own copies done, then wait until every rank is done reading the posted buffers
  mpr_status finish(cudaStream_t st) {
    mpr_status s = cuda(cudaStreamSynchronize(st), "group: stream sync");
    mpr_status b = barrier();
    return s != MPR_OK ? s : b;
  }

  template <class T>
  static void reduce_into(T* acc, const T* v, size_t n, CommOp op) {
    for (size_t i = 0; i < n; ++i) {
      if (op == OP_SUM) acc[i] = static_cast<T>(acc[i] + v[i]);
      else if (op == OP_MIN) acc[i] = v[i] < acc[i] ? v[i] : acc[i];
      else acc[i] = v[i] > acc[i] ? v[i] : acc[i];
    }
  }

  mpr_status allreduce(void* buf, size_t count, CommType t, CommOp op, cudaStream_t st) override {
    if (count == 0 || world == 1) return MPR_OK;
    const size_t es = comm_type_size(t), bytes = count * es;
    mpr_status s = publish(buf, count, st);
    if (s != MPR_OK) return s;
    // every rank reduces all contributions itself, in rank order (exact for integers)
    std::vector<char> all(bytes * world);
    for (int w = 0; w < world && s == MPR_OK; ++w)
      s = cuda(cudaMemcpyAsync(all.data() + w * bytes, g->post[w].ptr, bytes, cudaMemcpyDefault, st), "group: read");
    mpr_status f = finish(st);  // every rank has read every buffer before anyone writes
    if (s != MPR_OK) return s;
    if (f != MPR_OK) return f;
    char* acc = all.data();
    for (int w = 1; w < world; ++w) {
      const char* v = all.data() + w * bytes;
      switch (t) {
        case CT_U8: reduce_into(reinterpret_cast<uint8_t*>(acc), reinterpret_cast<const uint8_t*>(v), count, op); break;
        case CT_I32: reduce_into(reinterpret_cast<int32_t*>(acc), reinterpret_cast<const int32_t*>(v), count, op); break;
        case CT_I64: {  // two's-complement wrap-around like NCCL's int64 sum
          auto* a = reinterpret_cast<uint64_t*>(acc);
          const auto* b = reinterpret_cast<const uint64_t*>(v);
          if (op == OP_SUM) for (size_t i = 0; i < count; ++i) a[i] += b[i];
          else reduce_into(reinterpret_cast<int64_t*>(acc), reinterpret_cast<const int64_t*>(v), count, op);
          break;
        }
        case CT_U64: reduce_into(reinterpret_cast<uint64_t*>(acc), reinterpret_cast<const uint64_t*>(v), count, op); break;
        case CT_F32: reduce_into(reinterpret_cast<float*>(acc), reinterpret_cast<const float*>(v), count, op); break;
        case CT_F64: reduce_into(reinterpret_cast<double*>(acc), reinterpret_cast<const double*>(v), count, op); break;
      }
    }
    s = cuda(cudaMemcpyAsync(buf, acc, bytes, cudaMemcpyHostToDevice, st), "group: write");
    if (s != MPR_OK) return s;
    return cuda(cudaStreamSynchronize(st), "group: stream sync");
  }

  // Point to point, with NCCL's group semantics: every send of the call is posted first,
  // then every receive waits for its message and copies it, then the call returns once the
  // peers have copied this rank's sends (the buffers may be reused).
  mpr_status exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, CommType t,
                      cudaStream_t st) override {
    if (sends.empty() && recvs.empty()) return MPR_OK;
    const size_t es = comm_type_size(t);
    mpr_status s = cuda(cudaStreamSynchronize(st), "group: stream sync");
    if (s != MPR_OK) return s;
    std::vector<mpr_group::Msg*> mine;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (const P2P& p : sends) {
        if (p.peer < 0 || p.peer >= world) { err = "group: bad peer"; return MPR_ERR_INVALID_ARG; }
        const uint64_t seq = g->send_seq[static_cast<size_t>(rank * world + p.peer)]++;
        g->msgs.push_back({rank, p.peer, seq, p.ptr, p.count * es, false});
        mine.push_back(&g->msgs.back());
      }
      g->cv.notify_all();
    }
    for (const P2P& r : recvs) {
      if (r.peer < 0 || r.peer >= world) { err = "group: bad peer"; s = MPR_ERR_INVALID_ARG; break; }
      mpr_group::Msg* m = nullptr;
      {
        std::unique_lock<std::mutex> lk(g->mu);
        const uint64_t seq = g->recv_seq[static_cast<size_t>(r.peer * world + rank)]++;
        auto find = [&] {
          for (auto& x : g->msgs)
            if (x.src == r.peer && x.dst == rank && x.seq == seq) { m = &x; return true; }
          return false;
        };
        s = wait_for(lk, find, "a message from a peer");
        if (s != MPR_OK) break;
      }
      if (m->bytes != r.count * es) { err = "group: mis-sized receive"; s = MPR_ERR_STATE; }
      if (s == MPR_OK && m->bytes)
        s = cuda(cudaMemcpyAsync(r.ptr, m->ptr, m->bytes, cudaMemcpyDefault, st), "group: copy");
      if (s == MPR_OK) s = cuda(cudaStreamSynchronize(st), "group: stream sync");
      {
        std::lock_guard<std::mutex> lk(g->mu);
        m->done = true;  // consumed (even on error, so the sender does not wait forever)
        g->cv.notify_all();
      }
      if (s != MPR_OK) break;
    }
    {
      std::unique_lock<std::mutex> lk(g->mu);
      mpr_status w = wait_for(lk, [&] {
        for (auto* m : mine) if (!m->done) return false;
        return true;
      }, "the peers to receive");
      if (w == MPR_OK)
        g->msgs.remove_if([&](const mpr_group::Msg& x) {
          for (auto* m : mine) if (m == &x) return true;
          return false;
        });
      if (s == MPR_OK) s = w;
    }
    return s;
  }

  mpr_status allgatherv(const void* send, void* recv, const std::vector<size_t>& counts,
                        const std::vector<size_t>& displs, CommType t, cudaStream_t st) override {
    const size_t es = comm_type_size(t);
    char* r = static_cast<char*>(recv);
    if (world == 1) {
      if (send != r + displs[0] * es && counts[0])
        return cuda(cudaMemcpyAsync(r + displs[0] * es, send, counts[0] * es, cudaMemcpyDeviceToDevice, st), "copy");
      return MPR_OK;
    }
    mpr_status s = publish(send, counts[rank], st);
    if (s != MPR_OK) return s;
    for (int w = 0; w < world && s == MPR_OK; ++w) {
      char* dst = r + displs[w] * es;
      if (counts[w] && dst != g->post[w].ptr)
        s = cuda(cudaMemcpyAsync(dst, g->post[w].ptr, counts[w] * es, cudaMemcpyDefault, st), "group: gather");
    }
    mpr_status f = finish(st);
    return s != MPR_OK ? s : f;
  }

  mpr_status broadcast(void* buf, size_t count, CommType t, int root, cudaStream_t st) override {
    if (count == 0 || world == 1) return MPR_OK;
    mpr_status s = publish(buf, count, st);
    if (s != MPR_OK) return s;
    if (rank != root)
      s = cuda(cudaMemcpyAsync(buf, g->post[root].ptr, count * comm_type_size(t), cudaMemcpyDefault, st),
               "group: broadcast");
    mpr_status f = finish(st);
    return s != MPR_OK ? s : f;
  }
};

}  // namespace

Comm* make_nccl_comm(void* nccl_comm, int device, std::string& why) {
  if (!nccl().ok) {
    why = nccl().why;
    return nullptr;
  }
  auto* c = new NcclComm();
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  int n = 0, r = 0, d = -1;
  if (nccl().CommCount(c->comm, &n) != ncclSuccess || nccl().CommUserRank(c->comm, &r) != ncclSuccess ||
      nccl().CommCuDevice(c->comm, &d) != ncclSuccess) {
    why = "nccl_comm: cannot query the communicator";
    delete c;
    return nullptr;
  }
  if (d != device) {
    why = "nccl_comm lives on device " + std::to_string(d) + ", the context on " + std::to_string(device);
    delete c;
    return nullptr;
  }
  c->world = n;
  c->rank = r;
  return c;
}

Comm* make_group_comm(mpr_group* g, int rank, std::string& why) {
  if (!g || rank < 0 || rank >= g->world) {
    why = "group_rank must be in [0, world)";
    return nullptr;
  }
  auto* c = new GroupComm();
  c->g = g;
  c->rank = rank;
  c->world = g->world;
  return c;
}

mpr_status nccl_unique_id(void* id_out, std::string& why) {
  if (!nccl().ok) { why = nccl().why; return MPR_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) { why = nccl().GetErrorString(r); return MPR_ERR_NCCL; }
  std::memcpy(id_out, &id, sizeof id);
  return MPR_OK;
}

mpr_status nccl_comm_init(int world, int rank, const void* id, int device, void** comm_out, std::string& why) {
  if (!nccl().ok) { why = nccl().why; return MPR_ERR_NCCL; }
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) { why = "bad device"; return MPR_ERR_INVALID_ARG; }
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t comm = nullptr;
  ncclResult_t r = nccl().CommInitRank(&comm, world, u, rank);
  if (prev >= 0) cudaSetDevice(prev);
  if (r != ncclSuccess) { why = nccl().GetErrorString(r); return MPR_ERR_NCCL; }
  *comm_out = comm;
  return MPR_OK;
}

mpr_status nccl_comm_destroy(void* comm) {
  if (!comm || !nccl().ok) return MPR_OK;
  return nccl().CommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? MPR_OK : MPR_ERR_NCCL;
}

}  // namespace mpr

// ---- group lifecycle (C-ABI, declared in mpr.h)
extern "C" {
mpr_status mpr_group_create(int world, mpr_group** out) {
  if (!out || world < 1) return MPR_ERR_INVALID_ARG;
  auto* g = new mpr_group();
  g->world = world;
  g->post.resize(static_cast<size_t>(world));
  g->send_seq.assign(static_cast<size_t>(world) * world, 0);
  g->recv_seq.assign(static_cast<size_t>(world) * world, 0);
  *out = g;
  return MPR_OK;
}

void mpr_group_destroy(mpr_group* g) { delete g; }

mpr_status mpr_nccl_unique_id(void* id_out) {
  if (!id_out) return MPR_ERR_INVALID_ARG;
  std::string why;
  return mpr::nccl_unique_id(id_out, why);
}

mpr_status mpr_nccl_comm_init(int world, int rank, const void* id, int device, void** comm_out) {
  if (!id || !comm_out || world < 1 || rank < 0 || rank >= world) return MPR_ERR_INVALID_ARG;
  std::string why;
  mpr_status s = mpr::nccl_comm_init(world, rank, id, device, comm_out, why);
  return s;
}

mpr_status mpr_nccl_comm_destroy(void* comm) { return mpr::nccl_comm_destroy(comm); }
}
