// tls_comm.h — the exchange steps of the sharded path: in-place sum all-reduces
// of small fp64 buffers (dot-product partials, coarse coefficients) and point-to-point exchanges
// of halo rows (SpMV / overlap gathers) and of ASM overlap contributions (reverse halo) between
// the ranks that own disjoint row ranges / subdomain slabs.
//
//  * NcclComm   — one process per GPU; NCCL (libnccl.so.2, dlopen'ed so the library also loads on
//                 hosts without NCCL) over NVLink/NVSwitch; stream-ordered and CUDA-graph
//                 capturable, so the all-reduces live inside the replayed PCG/GMRES graphs.
//  * GroupComm  — R ranks inside ONE process on one device (host threads + stream events + a
//                 fixed-order sum kernel).  Used to validate the sharded schedule end-to-end on a
//                 single GPU; never spins on device flags (kernels only start after their stream
//                 waits are satisfied), not capturable (host barrier per reduction).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

namespace tls {

constexpr int MAX_GROUP = 16;

// One point-to-point exchange pattern: this rank sends sbuf[soff[k], +scnt[k]) to peers[k] and
// receives rbuf[roff[k], +rcnt[k]) from peers[k] (same peer list on both sides, ascending).
struct XPlan {
  std::vector<int> peers, scnt, rcnt;
  std::vector<long long> soff, roff;
  long long stot = 0, rtot = 0;
  int* d_sidx = nullptr;   // pack: sbuf[p] = src[d_sidx[p]]
  int* d_ridx = nullptr;   // unpack: dst[d_ridx[p]] = rbuf[p]
  double *sbuf = nullptr, *rbuf = nullptr;
  bool empty() const { return peers.empty(); }
};

struct Comm {
  int rank = 0, nranks = 1;
  long long calls[3] = {0, 0, 0};  // all-reduces, exchanges, all-gathers issued (tls_comm_info)
  virtual ~Comm() {}
  virtual int kind() const = 0;    // 1 NCCL, 2 in-process group, 3 recording
  virtual cudaError_t allreduce_sum(double* buf, long long count, cudaStream_t s, std::string& err) = 0;
  virtual cudaError_t exchange(const XPlan& x, cudaStream_t s, std::string& err) = 0;
  // recv[q * count + i] = send of rank q [i], i < count (every rank sends `count` doubles)
  virtual cudaError_t allgather(const double* send, long long count, double* recv, cudaStream_t s,
                                std::string& err) = 0;
  virtual bool capturable() const = 0;
};

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("dlopen libnccl.so.2: ") + dlerror();
      return false;
    }
    get_id = (decltype(get_id))dlsym(h, "ncclGetUniqueId");
    init_rank = (decltype(init_rank))dlsym(h, "ncclCommInitRank");
    allreduce = (decltype(allreduce))dlsym(h, "ncclAllReduce");
    allgather = (decltype(allgather))dlsym(h, "ncclAllGather");
    destroy = (decltype(destroy))dlsym(h, "ncclCommDestroy");
    errstr = (decltype(errstr))dlsym(h, "ncclGetErrorString");
    send = (decltype(send))dlsym(h, "ncclSend");
    recv = (decltype(recv))dlsym(h, "ncclRecv");
    group_start = (decltype(group_start))dlsym(h, "ncclGroupStart");
    group_end = (decltype(group_end))dlsym(h, "ncclGroupEnd");
    if (!get_id || !init_rank || !allreduce || !allgather || !destroy || !errstr || !send || !recv || !group_start ||
        !group_end) {
      err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    return true;
  }
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  return api;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl_api().destroy(comm);
  }
  int kind() const override { return 1; }
  cudaError_t allreduce_sum(double* buf, long long count, cudaStream_t s, std::string& err) override {
    ++calls[0];
    ncclResult_t r = nccl_api().allreduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, comm, s);
    if (r != ncclSuccess) {
      err = std::string("ncclAllReduce: ") + nccl_api().errstr(r);
      return cudaErrorUnknown;
    }
    return cudaSuccess;
  }
  // grouped send/recv with every peer of the plan (one NCCL group = one fused launch)
  cudaError_t exchange(const XPlan& x, cudaStream_t s, std::string& err) override {
    NcclApi& api = nccl_api();
    ++calls[1];
    ncclResult_t r = api.group_start();
    for (size_t k = 0; k < x.peers.size() && r == ncclSuccess; ++k) {
      if (x.scnt[k] > 0) r = api.send(x.sbuf + x.soff[k], (size_t)x.scnt[k], ncclFloat64, x.peers[k], comm, s);
      if (r == ncclSuccess && x.rcnt[k] > 0)
        r = api.recv(x.rbuf + x.roff[k], (size_t)x.rcnt[k], ncclFloat64, x.peers[k], comm, s);
    }
    ncclResult_t r2 = api.group_end();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
      err = std::string("ncclSend/ncclRecv: ") + api.errstr(r);
      return cudaErrorUnknown;
    }
    return cudaSuccess;
  }
  cudaError_t allgather(const double* send, long long count, double* recv, cudaStream_t s,
                        std::string& err) override {
    ++calls[2];
    ncclResult_t r = nccl_api().allgather(send, recv, (size_t)count, ncclFloat64, comm, s);
    if (r != ncclSuccess) {
      err = std::string("ncclAllGather: ") + nccl_api().errstr(r);
      return cudaErrorUnknown;
    }
    return cudaSuccess;
  }
  bool capturable() const override { return true; }
};

// ---------------------------------------------------------------- recording (tests)
// Capturable stand-in that moves no data and logs every collective the schedule issues
// (kind, element count, peers): lets a single-GPU test capture the sharded PCG / GMRES graphs
// exactly as the NCCL transport would and compare the per-rank collective sequences.
struct RecordComm : Comm {
  std::vector<long long> log;  // triples: kind (1 all-reduce, 2 exchange, 3 all-gather), count, peers
  int kind() const override { return 3; }
  cudaError_t allreduce_sum(double*, long long count, cudaStream_t, std::string&) override {
    log.insert(log.end(), {1LL, count, 0LL});
    return cudaSuccess;
  }
  cudaError_t exchange(const XPlan& x, cudaStream_t, std::string&) override {
    log.insert(log.end(), {2LL, x.stot + x.rtot, (long long)x.peers.size()});
    return cudaSuccess;
  }
  cudaError_t allgather(const double*, long long count, double*, cudaStream_t, std::string&) override {
    log.insert(log.end(), {3LL, count, 0LL});
    return cudaSuccess;
  }
  bool capturable() const override { return true; }
};

// ---------------------------------------------------------------- in-process group
struct GroupPtrs {
  const double* p[MAX_GROUP];
};

__global__ void k_group_sum(GroupPtrs ptrs, int n, long long count, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += ptrs.p[r][i];  // fixed rank order -> deterministic
    out[i] = s;
  }
}

struct GroupShared {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<double*> bufs;
  std::vector<cudaEvent_t> ev_in, ev_out;
  std::vector<const double*> xbuf;          // exchange: every member's send buffer
  std::vector<std::vector<long long>> xoff; // xoff[p][q]: offset of p's segment for q (-1: none)
  explicit GroupShared(int n_)
      : n(n_), bufs(n_, nullptr), ev_in(n_, nullptr), ev_out(n_, nullptr), xbuf(n_, nullptr),
        xoff(n_, std::vector<long long>(n_, -1)) {}
  bool broken = false;
  // false when a peer never arrives (it failed before reaching the exchange): the group is
  // then broken and every later exchange fails fast instead of hanging the process.
  bool barrier(int timeout_s = 120) {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct GroupComm : Comm {
  GroupShared* g = nullptr;
  double* tmp = nullptr;
  long long tmp_cap = 0;
  ~GroupComm() override {
    if (tmp) cudaFree(tmp);
  }
  int kind() const override { return 2; }
  cudaError_t allreduce_sum(double* buf, long long count, cudaStream_t s, std::string& err) override {
    cudaError_t e;
    if (count > tmp_cap) {
      if (tmp) cudaFree(tmp);
      if ((e = cudaMalloc((void**)&tmp, sizeof(double) * count)) != cudaSuccess) return e;
      tmp_cap = count;
    }
    g->bufs[rank] = buf;
    if ((e = cudaEventRecord(g->ev_in[rank], s)) != cudaSuccess) return e;
    if (!g->barrier()) {  // every member's partial is enqueued
      err = "in-process group: a peer rank did not reach the exchange";
      return cudaErrorUnknown;
    }
    GroupPtrs ptrs{};
    for (int r = 0; r < g->n; ++r) {
      if ((e = cudaStreamWaitEvent(s, g->ev_in[r], 0)) != cudaSuccess) return e;
      ptrs.p[r] = g->bufs[r];
    }
    const int grid = (int)std::min<long long>((count + 255) / 256, 1184);
    k_group_sum<<<grid > 0 ? grid : 1, 256, 0, s>>>(ptrs, g->n, count, tmp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaEventRecord(g->ev_out[rank], s)) != cudaSuccess) return e;
    if (!g->barrier()) {  // every member has enqueued its reads of all partials
      err = "in-process group: a peer rank did not reach the exchange";
      return cudaErrorUnknown;
    }
    for (int r = 0; r < g->n; ++r)
      if ((e = cudaStreamWaitEvent(s, g->ev_out[r], 0)) != cudaSuccess) return e;
    return cudaMemcpyAsync(buf, tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, s);
  }
  // every member publishes its send buffer; each copies its segments out of the peers' buffers
  cudaError_t exchange(const XPlan& x, cudaStream_t s, std::string& err) override {
    cudaError_t e;
    std::fill(g->xoff[rank].begin(), g->xoff[rank].end(), -1LL);
    for (size_t k = 0; k < x.peers.size(); ++k) g->xoff[rank][x.peers[k]] = x.scnt[k] > 0 ? x.soff[k] : -1;
    g->xbuf[rank] = x.sbuf;
    if ((e = cudaEventRecord(g->ev_in[rank], s)) != cudaSuccess) return e;
    if (!g->barrier()) {
      err = "in-process group: a peer rank did not reach the exchange";
      return cudaErrorUnknown;
    }
    for (size_t k = 0; k < x.peers.size(); ++k) {
      if (x.rcnt[k] == 0) continue;
      const int p = x.peers[k];
      if (g->xoff[p][rank] < 0) {
        err = "in-process group: exchange plans disagree";
        return cudaErrorUnknown;
      }
      if ((e = cudaStreamWaitEvent(s, g->ev_in[p], 0)) != cudaSuccess) return e;
      if ((e = cudaMemcpyAsync(x.rbuf + x.roff[k], g->xbuf[p] + g->xoff[p][rank], sizeof(double) * x.rcnt[k],
                               cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return e;
    }
    if ((e = cudaEventRecord(g->ev_out[rank], s)) != cudaSuccess) return e;
    if (!g->barrier()) {  // every member has enqueued its reads of the send buffers
      err = "in-process group: a peer rank did not reach the exchange";
      return cudaErrorUnknown;
    }
    for (int r = 0; r < g->n; ++r)
      if ((e = cudaStreamWaitEvent(s, g->ev_out[r], 0)) != cudaSuccess) return e;
    return cudaSuccess;
  }
  // every member publishes its send buffer; each copies all of them, in rank order
  cudaError_t allgather(const double* send, long long count, double* recv, cudaStream_t s,
                        std::string& err) override {
    cudaError_t e;
    g->xbuf[rank] = send;
    if ((e = cudaEventRecord(g->ev_in[rank], s)) != cudaSuccess) return e;
    if (!g->barrier()) {
      err = "in-process group: a peer rank did not reach the all-gather";
      return cudaErrorUnknown;
    }
    for (int r = 0; r < g->n; ++r) {
      if ((e = cudaStreamWaitEvent(s, g->ev_in[r], 0)) != cudaSuccess) return e;
      if ((e = cudaMemcpyAsync(recv + (long long)r * count, g->xbuf[r], sizeof(double) * count,
                               cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return e;
    }
    if ((e = cudaEventRecord(g->ev_out[rank], s)) != cudaSuccess) return e;
    if (!g->barrier()) {
      err = "in-process group: a peer rank did not reach the all-gather";
      return cudaErrorUnknown;
    }
    for (int r = 0; r < g->n; ++r)
      if ((e = cudaStreamWaitEvent(s, g->ev_out[r], 0)) != cudaSuccess) return e;
    return cudaSuccess;
  }
  bool capturable() const override { return false; }
};

}  // namespace tls
