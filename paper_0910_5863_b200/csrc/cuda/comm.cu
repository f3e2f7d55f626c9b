// Exchange layer of the sharded engine (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../host/host.hpp"
#include "dense.cuh"
#include "devbuf.cuh"

namespace b200 {

double Comm::max_all(double v) {
  std::vector<char> mine(sizeof(double));
  std::memcpy(mine.data(), &v, sizeof(double));
  double m = v;
  for (const auto& b : allgather(mine)) {
    double x;
    std::memcpy(&x, b.data(), sizeof(double));
    m = x > m ? x : m;
  }
  return m;
}

// ---------------------------------------------------------------------------
// loopback: ranks are host threads of one process
// ---------------------------------------------------------------------------
namespace {
struct LoopGroup {
  std::mutex mu;
  std::condition_variable cv;
  int world = 0, arrived = 0;
  long long generation = 0;
  std::vector<std::vector<char>> slots;

  // every rank deposits `mine`; returns all deposits in rank order
  std::vector<std::vector<char>> exchange(int rank, const std::vector<char>& mine) {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    slots[rank] = mine;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
    std::vector<std::vector<char>> out = slots;
    // second barrier: nobody overwrites a slot before everyone has copied them
    const long long gen2 = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen2; });
    }
    return out;
  }
};

std::mutex g_groups_mu;
std::map<int, std::shared_ptr<LoopGroup>> g_groups;

class LoopbackComm : public Comm {
 public:
  LoopbackComm(std::shared_ptr<LoopGroup> g, int rank) : g_(std::move(g)), rank_(rank) {
    if (g_->world > 1) shared_device_users(+1);  // the ranks' engines launch concurrently on one GPU
  }
  ~LoopbackComm() override {
    if (g_->world > 1) shared_device_users(-1);
  }
  int rank() const override { return rank_; }
  int world() const override { return g_->world; }
  void allreduce(double* d, std::size_t n, cudaStream_t st) override {
    std::vector<char> mine(n * sizeof(double));
    if (n) CK(cudaMemcpyAsync(mine.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const auto all = g_->exchange(rank_, mine);
    std::vector<double> sum(n, 0.0);
    for (const auto& b : all) {  // rank order: identical on every rank
      const double* x = reinterpret_cast<const double*>(b.data());
      for (std::size_t i = 0; i < n; ++i) sum[i] += x[i];
    }
    if (n) CK(cudaMemcpyAsync(d, sum.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  std::vector<std::vector<char>> allgather(const std::vector<char>& mine) override {
    return g_->exchange(rank_, mine);
  }
  void exchange(const std::vector<Segment>& sends, const std::vector<Segment>& recvs, cudaStream_t st) override {
    // one blob per rank: [peer, n, n doubles]... ; every rank reads the
    // messages addressed to it from each peer's blob, in order
    std::vector<char> mine;
    for (const Segment& sg : sends) {
      const long long hdr[2] = {sg.peer, static_cast<long long>(sg.n)};
      const std::size_t at = mine.size();
      mine.resize(at + sizeof(hdr) + sg.n * sizeof(double));
      std::memcpy(mine.data() + at, hdr, sizeof(hdr));
      if (sg.n)
        CK(cudaMemcpyAsync(mine.data() + at + sizeof(hdr), sg.ptr, sg.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    const auto all = g_->exchange(rank_, mine);
    std::vector<std::size_t> cursor(all.size(), 0);
    for (const Segment& rv : recvs) {
      const auto& b = all.at(rv.peer);
      std::size_t& c = cursor[rv.peer];
      for (;;) {  // next message of that peer addressed to this rank
        if (c >= b.size()) throw Error(kError, "loopback exchange: missing message");
        long long hdr[2];
        std::memcpy(hdr, b.data() + c, sizeof(hdr));
        const std::size_t body = c + sizeof(hdr);
        c = body + static_cast<std::size_t>(hdr[1]) * sizeof(double);
        if (hdr[0] != rank_) continue;
        if (static_cast<std::size_t>(hdr[1]) != rv.n) throw Error(kError, "loopback exchange: size mismatch");
        if (rv.n) CK(cudaMemcpyAsync(rv.ptr, b.data() + body, rv.n * sizeof(double), cudaMemcpyHostToDevice, st));
        break;
      }
    }
    CK(cudaStreamSynchronize(st));
  }

 private:
  std::shared_ptr<LoopGroup> g_;
  int rank_;
};
}  // namespace

std::shared_ptr<Comm> make_loopback_comm(int group, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(kError, "loopback: bad rank/world");
  std::lock_guard<std::mutex> lk(g_groups_mu);
  auto& g = g_groups[group];
  if (!g || g->world != world) {
    g = std::make_shared<LoopGroup>();
    g->world = world;
    g->slots.assign(world, {});
  }
  return std::make_shared<LoopbackComm>(g, rank);
}

// ---------------------------------------------------------------------------
// NCCL (resolved at run time: the process may already hold torch's libnccl)
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(kCudaError, "NCCL library not found (libnccl.so.2)");
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw Error(kCudaError, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  loaded = true;
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(kCudaError, std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

class NcclComm : public Comm {
 public:
  NcclComm(const unsigned char* id, int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    nck(nccl().CommInitRank(&comm_, world, uid, rank), "CommInitRank");
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
    if (st_) cudaStreamDestroy(st_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void allreduce(double* d, std::size_t n, cudaStream_t st) override {
    if (world_ > 1 && n) nck(nccl().AllReduce(d, d, n, ncclDouble, ncclSum, comm_, st), "AllReduce");
  }
  void exchange(const std::vector<Segment>& sends, const std::vector<Segment>& recvs, cudaStream_t st) override {
    if (sends.empty() && recvs.empty()) return;
    nck(nccl().GroupStart(), "GroupStart");
    for (const Segment& sg : sends)
      if (sg.n) nck(nccl().Send(sg.ptr, sg.n, ncclDouble, sg.peer, comm_, st), "Send");
    for (const Segment& rv : recvs)
      if (rv.n) nck(nccl().Recv(rv.ptr, rv.n, ncclDouble, rv.peer, comm_, st), "Recv");
    nck(nccl().GroupEnd(), "GroupEnd");
  }
  std::vector<std::vector<char>> allgather(const std::vector<char>& mine) override {
    // sizes first, then the blobs padded to the largest
    std::vector<long long> sizes(world_);
    size_buf_.alloc(world_ + 1);
    long long n = static_cast<long long>(mine.size());
    CK(cudaMemcpyAsync(size_buf_.p + world_, &n, sizeof(n), cudaMemcpyHostToDevice, st_));
    nck(nccl().AllGather(size_buf_.p + world_, size_buf_.p, 1, ncclInt64, comm_, st_), "AllGather");
    CK(cudaMemcpyAsync(sizes.data(), size_buf_.p, world_ * sizeof(long long), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    long long mx = 1;
    for (long long s : sizes) mx = s > mx ? s : mx;
    blob_.alloc(static_cast<std::size_t>(mx) * (world_ + 1));
    char* send = blob_.p + static_cast<std::size_t>(mx) * world_;
    if (n) CK(cudaMemcpyAsync(send, mine.data(), n, cudaMemcpyHostToDevice, st_));
    nck(nccl().AllGather(send, blob_.p, static_cast<std::size_t>(mx), ncclChar, comm_, st_), "AllGather");
    std::vector<char> all(static_cast<std::size_t>(mx) * world_);
    CK(cudaMemcpyAsync(all.data(), blob_.p, all.size(), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    std::vector<std::vector<char>> out(world_);
    for (int r = 0; r < world_; ++r)
      out[r].assign(all.begin() + static_cast<std::size_t>(mx) * r, all.begin() + static_cast<std::size_t>(mx) * r + sizes[r]);
    return out;
  }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
  cudaStream_t st_ = nullptr;
  DBuf<long long> size_buf_;
  DBuf<char> blob_;
};
}  // namespace

void nccl_unique_id(unsigned char* id) {
  ncclUniqueId uid;
  nck(nccl().GetUniqueId(&uid), "GetUniqueId");
  std::memcpy(id, uid.internal, NCCL_UNIQUE_ID_BYTES);
}

std::shared_ptr<Comm> make_nccl_comm(const unsigned char* id, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(kError, "nccl: bad rank/world");
  return std::make_shared<NcclComm>(id, rank, world);
}

}  // namespace b200
