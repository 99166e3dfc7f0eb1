// Multi-GPU halo layer of libfastilu_b200.
//
// Rank p owns contiguous global rows.  Its local layout is [G ghost rows | n owned rows] with
// extended vectors [G | n | H].  Per sweep, rank p-1 sends the whole stored rows (values and
// diagonal copies) of the G_p rows rank p reads, as ONE contiguous range on both sides (same
// exact pattern on both ranks, so no pack/unpack).  Trisolve halos: z (lower, from p-1) and
// w (upper, from p+1).  Two transports:
//   FASTILU_COMM_NCCL  : ncclSend/ncclRecv pairs in a group on the handle's stream (NCCL is
//                        dlopen'ed, so single-GPU use never needs it);
//   FASTILU_COMM_LOCAL : ranks are threads of one process (same or different devices);
//                        device-to-device copies ordered by events, host barriers between.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "comm.h"

#define FAIL(code)                                                                  \
  do {                                                                              \
    if (std::getenv("FASTILU_DEBUG"))                                               \
      fprintf(stderr, "fastilu: %s at %s:%d\n", #code, __FILE__, __LINE__);         \
    return code;                                                                    \
  } while (0)

struct fastilu_group_s {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  // publication slots (one per rank)
  std::vector<const void *> ptr;
  std::vector<cudaEvent_t> ev;
  std::vector<std::vector<int64_t>> ints;
  std::vector<std::vector<double>> dbl;
  std::vector<int> dev;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    int64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      generation++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

extern "C" fastilu_status fastilu_group_create(fastilu_group *out, int nranks) {
  if (!out || nranks < 1) FAIL(FASTILU_ERR_INVALID_ARG);
  fastilu_group g = new (std::nothrow) fastilu_group_s();
  if (!g) return FASTILU_ERR_OOM;
  g->nranks = nranks;
  g->ptr.assign(nranks, nullptr);
  g->ev.assign(nranks, nullptr);
  g->ints.assign(nranks, {});
  g->dbl.assign(nranks, {});
  g->dev.assign(nranks, 0);
  *out = g;
  return FASTILU_OK;
}

extern "C" fastilu_status fastilu_group_destroy(fastilu_group g) {
  delete g;
  return FASTILU_OK;
}

namespace fastilu {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

static NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define LD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    LD(GetUniqueId);
    LD(CommInitRank);
    LD(CommDestroy);
    LD(Send);
    LD(Recv);
    LD(AllGather);
    LD(AllReduce);
    LD(GroupStart);
    LD(GroupEnd);
#undef LD
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
             api.AllGather && api.AllReduce && api.GroupStart && api.GroupEnd;
  });
  return api;
}

struct Comm {
  int kind = FASTILU_COMM_NONE;
  int rank = 0, nranks = 1, dev = 0;
  fastilu_group grp = nullptr;
  ncclComm_t nc = nullptr;
  // partition of every rank: row_begin, n, G, H, tail-count, ghost-count
  std::vector<int64_t> rb, nn, GG, HH;
  int64_t G = 0, H = 0, n = 0;
  // factor halo ranges (elements of vals): what I send to p+1, what I receive from p-1
  int64_t send_off = 0, send_cnt = 0, recv_cnt = 0;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  int64_t *d_scratch = nullptr;  // NCCL setup / reductions
  size_t scratch_elems = 0;
  cudaStream_t host_stream = nullptr;  // host-side reductions (created once, NCCL only)
  // packed factor halo (template layout), overlapped with the interior sweep
  cudaStream_t halo_stream = nullptr;
  cudaEvent_t ev_src = nullptr, ev_halo = nullptr;
  double *d_hsend = nullptr, *d_hrecv = nullptr;
  int64_t hsend_cap = 0, hrecv_cap = 0;
};

#define CUC(x)                                                    \
  do {                                                            \
    if ((x) != cudaSuccess) return FASTILU_ERR_CUDA;              \
  } while (0)
#define NCC(x)                                                    \
  do {                                                            \
    if ((x) != ncclSuccess) FAIL(FASTILU_ERR_NCCL);              \
  } while (0)

static fastilu_status scratch(Comm *c, size_t elems) {
  if (c->scratch_elems >= elems) return FASTILU_OK;
  if (c->d_scratch) cudaFree(c->d_scratch);
  c->d_scratch = nullptr;
  CUC(cudaMalloc((void **)&c->d_scratch, elems * sizeof(int64_t)));
  c->scratch_elems = elems;
  return FASTILU_OK;
}

// all-gather K int64 per rank (host in, host out [nranks][K])
static fastilu_status allgather_i64(Comm *c, const std::vector<int64_t> &mine,
                                    std::vector<int64_t> &all, cudaStream_t st) {
  const size_t K = mine.size();
  all.assign(K * c->nranks, 0);
  if (c->kind == FASTILU_COMM_LOCAL) {
    c->grp->ints[c->rank] = mine;
    c->grp->barrier();
    for (int r = 0; r < c->nranks; r++)
      std::memcpy(&all[r * K], c->grp->ints[r].data(), K * sizeof(int64_t));
    c->grp->barrier();
    return FASTILU_OK;
  }
  fastilu_status s = scratch(c, K * (c->nranks + 1));
  if (s) return s;
  CUC(cudaMemcpyAsync(c->d_scratch, mine.data(), K * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  NCC(nccl().AllGather(c->d_scratch, c->d_scratch + K, K, ncclInt64, c->nc, st));
  CUC(cudaMemcpyAsync(all.data(), c->d_scratch + K, K * c->nranks * sizeof(int64_t),
                      cudaMemcpyDeviceToHost, st));
  CUC(cudaStreamSynchronize(st));
  return FASTILU_OK;
}

fastilu_status comm_init(Comm *&out, const fastilu_options &o, cudaStream_t st) {
  out = nullptr;
  Comm *c = new (std::nothrow) Comm();
  if (!c) return FASTILU_ERR_OOM;
  out = c;
  c->kind = o.comm_kind;
  c->rank = o.rank;
  c->nranks = o.nranks;
  CUC(cudaGetDevice(&c->dev));
  if (c->kind == FASTILU_COMM_LOCAL) {
    if (!o.group || o.group->nranks != o.nranks) FAIL(FASTILU_ERR_INVALID_ARG);
    c->grp = o.group;
    c->grp->dev[c->rank] = c->dev;
  } else if (c->kind == FASTILU_COMM_NCCL) {
    if (!o.nccl_unique_id) FAIL(FASTILU_ERR_INVALID_ARG);
    if (!nccl().ok) FAIL(FASTILU_ERR_NCCL);
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_unique_id, sizeof(id));
    NCC(nccl().CommInitRank(&c->nc, o.nranks, id, o.rank));
    CUC(cudaStreamCreateWithFlags(&c->host_stream, cudaStreamNonBlocking));
  } else {
    FAIL(FASTILU_ERR_INVALID_ARG);
  }
  CUC(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  CUC(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  CUC(cudaEventCreateWithFlags(&c->ev_src, cudaEventDisableTiming));
  CUC(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  CUC(cudaStreamCreateWithFlags(&c->halo_stream, cudaStreamNonBlocking));
  (void)st;
  return FASTILU_OK;
}

fastilu_status comm_allgather_i64(Comm *c, const std::vector<int64_t> &mine,
                                  std::vector<int64_t> &all, cudaStream_t st) {
  return allgather_i64(c, mine, all, st);
}

fastilu_status comm_layout(Comm *c, int64_t row_begin, int64_t n, int64_t G, int64_t H,
                           const int64_t *h_rp, int64_t stat, int64_t *stat_global,
                           int tsell_W, uint64_t layout_hash, cudaStream_t st) {
  c->G = G;
  c->H = H;
  c->n = n;
  // partition exchange: row_begin, n, G, H, nnz of my trailing rows (by request), my ghost nnz
  std::vector<int64_t> all;
  fastilu_status s = allgather_i64(c, {row_begin, n, G, H}, all, st);
  if (s) return s;
  const int P = c->nranks, p = c->rank;
  c->rb.resize(P);
  c->nn.resize(P);
  c->GG.resize(P);
  c->HH.resize(P);
  for (int r = 0; r < P; r++) {
    c->rb[r] = all[4 * r];
    c->nn[r] = all[4 * r + 1];
    c->GG[r] = all[4 * r + 2];
    c->HH[r] = all[4 * r + 3];
  }
  for (int r = 0; r < P; r++) {
    if (r > 0 && c->rb[r] != c->rb[r - 1] + c->nn[r - 1]) FAIL(FASTILU_ERR_INVALID_ARG);
    if (r == 0 && c->GG[r] != 0) FAIL(FASTILU_ERR_INVALID_ARG);
    if (r == P - 1 && c->HH[r] != 0) FAIL(FASTILU_ERR_INVALID_ARG);
    // ghosts must come from the immediate neighbours only
    if (r > 0 && c->GG[r] > c->nn[r - 1]) FAIL(FASTILU_ERR_UNSUPPORTED);
    if (r < P - 1 && c->HH[r] > c->nn[r + 1]) FAIL(FASTILU_ERR_UNSUPPORTED);
  }
  // factor halo: I send my last G_{p+1} owned rows (local rows [G + n - G_{p+1}, G + n))
  const int64_t gn = (p + 1 < P) ? c->GG[p + 1] : 0;
  if (tsell_W > 0) {  // whole 32-row slices of the template layout (G, n multiples of 32)
    c->send_off = (G + n - gn) * (int64_t)tsell_W;
    c->send_cnt = gn * (int64_t)tsell_W;
    c->recv_cnt = G * (int64_t)tsell_W;
  } else {
    c->send_off = h_rp[G + n - gn];
    c->send_cnt = h_rp[G + n] - c->send_off;
    c->recv_cnt = h_rp[G];
  }
  s = allgather_i64(c, {c->send_cnt, c->recv_cnt, stat, (int64_t)layout_hash}, all, st);
  if (s) return s;
  for (int r = 0; r + 1 < P; r++)
    if (all[4 * r] != all[4 * (r + 1) + 1]) FAIL(FASTILU_ERR_BAD_MATRIX);  // patterns disagree
  for (int r = 0; r < P; r++)
    if (all[4 * r + 3] != all[3]) FAIL(FASTILU_ERR_UNSUPPORTED);  // layouts differ
  *stat_global = 0;
  for (int r = 0; r < P; r++) *stat_global += all[4 * r + 2];
  return FASTILU_OK;
}

// One exchange: up to two sends (to p+1, to p-1) and two receives, each a list of ranges.
struct Xfer {
  const double *src;
  double *dst;
  int64_t cnt;
  int peer;
};

static fastilu_status exchange(Comm *c, const std::vector<Xfer> &sends,
                               const std::vector<Xfer> &recvs, cudaStream_t st) {
  if (c->kind == FASTILU_COMM_NCCL) {
    NCC(nccl().GroupStart());
    for (const Xfer &x : sends)
      if (x.cnt > 0) NCC(nccl().Send(x.src, (size_t)x.cnt, ncclFloat64, x.peer, c->nc, st));
    for (const Xfer &x : recvs)
      if (x.cnt > 0) NCC(nccl().Recv(x.dst, (size_t)x.cnt, ncclFloat64, x.peer, c->nc, st));
    NCC(nccl().GroupEnd());
    return FASTILU_OK;
  }
  // LOCAL: receivers pull.  1) publish my send sources + ready event
  fastilu_group g = c->grp;
  CUC(cudaEventRecord(c->ev_ready, st));
  g->ev[c->rank] = c->ev_ready;
  g->barrier();
  // publish (source pointer) per destination through the int slots: [peer, ptr, cnt]...
  std::vector<int64_t> pub;
  for (const Xfer &x : sends) {
    pub.push_back(x.peer);
    pub.push_back((int64_t)(intptr_t)x.src);
    pub.push_back(x.cnt);
  }
  g->ints[c->rank] = pub;
  g->barrier();
  // 2) pull what my neighbours publish for me
  for (const Xfer &x : recvs) {
    const std::vector<int64_t> &q = g->ints[x.peer];
    const double *src = nullptr;
    int64_t cnt = -1;
    for (size_t i = 0; i + 2 < q.size(); i += 3)
      if (q[i] == c->rank) {
        src = (const double *)(intptr_t)q[i + 1];
        cnt = q[i + 2];
      }
    if (cnt != x.cnt) FAIL(FASTILU_ERR_STATE);
    if (cnt > 0) {
      CUC(cudaStreamWaitEvent(st, g->ev[x.peer], 0));
      if (g->dev[x.peer] == c->dev)
        CUC(cudaMemcpyAsync(x.dst, src, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
      else
        CUC(cudaMemcpyPeerAsync(x.dst, c->dev, src, g->dev[x.peer], cnt * sizeof(double), st));
    }
  }
  CUC(cudaEventRecord(c->ev_done, st));
  g->barrier();
  g->ev[c->rank] = c->ev_done;
  g->barrier();
  // 3) my sources may be overwritten only after my receivers' copies finished
  for (const Xfer &x : sends)
    if (x.cnt > 0) CUC(cudaStreamWaitEvent(st, g->ev[x.peer], 0));
  g->barrier();
  return FASTILU_OK;
}

fastilu_status comm_vector_halo(Comm *c, double *x, cudaStream_t st, bool lower, bool upper) {
  const int P = c->nranks, p = c->rank;
  std::vector<Xfer> sends, recvs;
  if (lower) {  // my last G_{p+1} owned entries -> p+1's [0, G_{p+1}); I receive [0, G)
    if (p + 1 < P) sends.push_back({x + c->G + c->n - c->GG[p + 1], nullptr, c->GG[p + 1], p + 1});
    if (p > 0) recvs.push_back({nullptr, x, c->G, p - 1});
  }
  if (upper) {  // my first H_{p-1} owned entries -> p-1's [G+n, G+n+H); I receive my H
    if (p > 0) sends.push_back({x + c->G, nullptr, c->HH[p - 1], p - 1});
    if (p + 1 < P) recvs.push_back({nullptr, x + c->G + c->n, c->H, p + 1});
  }
  return exchange(c, sends, recvs, st);
}

fastilu_status comm_vector_halo_async(Comm *c, double *x, cudaStream_t st, bool lower,
                                      bool upper, cudaEvent_t *done) {
  CUC(cudaEventRecord(c->ev_src, st));
  CUC(cudaStreamWaitEvent(c->halo_stream, c->ev_src, 0));
  fastilu_status s = comm_vector_halo(c, x, c->halo_stream, lower, upper);
  if (s) return s;
  CUC(cudaEventRecord(c->ev_halo, c->halo_stream));
  *done = c->ev_halo;
  return FASTILU_OK;
}

fastilu_status comm_factor_halo(Comm *c, double *vals, const int64_t *, double *udiag,
                                cudaStream_t st) {
  const int P = c->nranks, p = c->rank;
  std::vector<Xfer> sends, recvs;
  if (p + 1 < P) {
    sends.push_back({vals + c->send_off, nullptr, c->send_cnt, p + 1});
    sends.push_back({udiag + c->G + c->n - c->GG[p + 1], nullptr, c->GG[p + 1], p + 1});
  }
  if (p > 0) {
    recvs.push_back({nullptr, vals, c->recv_cnt, p - 1});
    recvs.push_back({nullptr, udiag, c->G, p - 1});
  }
  // LOCAL pulls match sends by (peer, order): publish both ranges in order
  if (c->kind == FASTILU_COMM_LOCAL) {
    // exchange() matches one range per peer; do two rounds
    std::vector<Xfer> s1, r1, s2, r2;
    for (size_t i = 0; i < sends.size(); i++) (i % 2 == 0 ? s1 : s2).push_back(sends[i]);
    for (size_t i = 0; i < recvs.size(); i++) (i % 2 == 0 ? r1 : r2).push_back(recvs[i]);
    fastilu_status s = exchange(c, s1, r1, st);
    if (s) return s;
    return exchange(c, s2, r2, st);
  }
  return exchange(c, sends, recvs, st);
}

fastilu_status comm_factor_halo_upper(Comm *c, double *vals, double *udiag, int W, int c0,
                                      cudaStream_t st, cudaEvent_t *done) {
  const int P = c->nranks, p = c->rank;
  const int64_t NC = W - c0;
  const int64_t gn = (p + 1 < P) ? c->GG[p + 1] : 0;  // owned rows rank p+1 keeps as ghosts
  if ((gn % 32) || (c->G % 32)) FAIL(FASTILU_ERR_UNSUPPORTED);
  const int64_t ns_send = gn / 32, ns_recv = c->G / 32;
  const int64_t cnt_send = ns_send * NC * 32, cnt_recv = ns_recv * NC * 32;
  if (cnt_send > c->hsend_cap) {
    if (c->d_hsend) cudaFree(c->d_hsend);
    c->d_hsend = nullptr;
    CUC(cudaMalloc((void **)&c->d_hsend, sizeof(double) * cnt_send));
    c->hsend_cap = cnt_send;
  }
  if (cnt_recv > c->hrecv_cap) {
    if (c->d_hrecv) cudaFree(c->d_hrecv);
    c->d_hrecv = nullptr;
    CUC(cudaMalloc((void **)&c->d_hrecv, sizeof(double) * cnt_recv));
    c->hrecv_cap = cnt_recv;
  }
  cudaStream_t hs = c->halo_stream;
  // the iterate is complete on the compute stream before it is packed
  CUC(cudaEventRecord(c->ev_src, st));
  CUC(cudaStreamWaitEvent(hs, c->ev_src, 0));
  if (ns_send)
    CUC(launch_tsell_pack_upper(vals, (c->G + c->n - gn) / 32, ns_send, W, c0, c->d_hsend, hs));
  std::vector<Xfer> sends, recvs;
  if (p + 1 < P) sends.push_back({c->d_hsend, nullptr, cnt_send, p + 1});
  if (p > 0) recvs.push_back({nullptr, c->d_hrecv, cnt_recv, p - 1});
  fastilu_status s = exchange(c, sends, recvs, hs);
  if (s) return s;
  if (ns_recv) CUC(launch_tsell_unpack_upper(c->d_hrecv, 0, ns_recv, W, c0, vals, udiag, hs));
  CUC(cudaEventRecord(c->ev_halo, hs));
  *done = c->ev_halo;
  return FASTILU_OK;
}

int64_t comm_halo_bytes(const Comm *c, int W, int c0) {
  const int P = c->nranks, p = c->rank;
  const int64_t gn = (p + 1 < P) ? c->GG[p + 1] : 0;
  return W > 0 ? gn * (int64_t)(W - c0) * 8 : c->send_cnt * 8;
}

fastilu_status comm_allreduce_host(Comm *c, double *r2, int count, ErrFlags &ef) {
  if (c->kind == FASTILU_COMM_LOCAL) {
    fastilu_group g = c->grp;
    std::vector<double> mine(r2, r2 + count);
    mine.push_back((double)0);
    g->dbl[c->rank] = mine;
    g->ints[c->rank] = {(int64_t)ef.zero_diag, (int64_t)ef.zero_pivot};
    g->barrier();
    for (int i = 0; i < count; i++) {
      double t = 0.0;
      for (int r = 0; r < c->nranks; r++) t += g->dbl[r][i];  // rank order: deterministic
      r2[i] = t;
    }
    unsigned long long zd = ~0ull, zp = ~0ull;
    for (int r = 0; r < c->nranks; r++) {
      zd = std::min(zd, (unsigned long long)g->ints[r][0]);
      zp = std::min(zp, (unsigned long long)g->ints[r][1]);
    }
    ef.zero_diag = zd;
    ef.zero_pivot = zp;
    g->barrier();
    return FASTILU_OK;
  }
  // NCCL: doubles summed, flags min-reduced (as uint64)
  fastilu_status s = scratch(c, (size_t)count + 2);
  if (s) return s;
  cudaStream_t st = c->host_stream;
  double *d = reinterpret_cast<double *>(c->d_scratch);
  uint64_t flags[2] = {ef.zero_diag, ef.zero_pivot};
  if (count) CUC(cudaMemcpyAsync(d, r2, count * sizeof(double), cudaMemcpyHostToDevice, st));
  CUC(cudaMemcpyAsync(c->d_scratch + count, flags, sizeof(flags), cudaMemcpyHostToDevice, st));
  NCC(nccl().GroupStart());
  if (count) NCC(nccl().AllReduce(d, d, count, ncclFloat64, ncclSum, c->nc, st));
  NCC(nccl().AllReduce(c->d_scratch + count, c->d_scratch + count, 2, ncclUint64, ncclMin, c->nc,
                       st));
  NCC(nccl().GroupEnd());
  if (count) CUC(cudaMemcpyAsync(r2, d, count * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUC(cudaMemcpyAsync(flags, c->d_scratch + count, sizeof(flags), cudaMemcpyDeviceToHost, st));
  CUC(cudaStreamSynchronize(st));
  ef.zero_diag = flags[0];
  ef.zero_pivot = flags[1];
  return FASTILU_OK;
}

void comm_destroy(Comm *c) {
  if (!c) return;
  if (c->nc && nccl().ok) nccl().CommDestroy(c->nc);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->d_scratch) cudaFree(c->d_scratch);
  if (c->host_stream) cudaStreamDestroy(c->host_stream);
  if (c->halo_stream) cudaStreamDestroy(c->halo_stream);
  if (c->ev_src) cudaEventDestroy(c->ev_src);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->d_hsend) cudaFree(c->d_hsend);
  if (c->d_hrecv) cudaFree(c->d_hrecv);
  delete c;
}

}  // namespace fastilu

extern "C" fastilu_status fastilu_nccl_unique_id(void *id128) {
  if (!id128) FAIL(FASTILU_ERR_INVALID_ARG);
  if (!fastilu::nccl().ok) FAIL(FASTILU_ERR_NCCL);
  ncclUniqueId id;
  if (fastilu::nccl().GetUniqueId(&id) != ncclSuccess) FAIL(FASTILU_ERR_NCCL);
  std::memcpy(id128, &id, sizeof(id));
  return FASTILU_OK;
}
