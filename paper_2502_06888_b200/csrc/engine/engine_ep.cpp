// SPDX-License-Identifier: Apache-2.0
// Expert parallelism for the B200 engine.
//
// Sharding: global expert e lives on rank e % G as local expert e / G; each
// rank holds (and streams over its own host link) only its E/G experts per
// layer, attention/router weights are replicated, and every rank runs
// attention + router for its own batch group (data parallel). Per layer:
//   1. router on own tokens (global ids), then on the compute stream:
//      - integer all-reduce of the expert histogram and of the
//        co-activation delta (so every rank keeps the identical global
//        correlation table the single-GPU prefetcher would), next-layer
//        prefetch scores;
//      - destination-major relabel (owner*E_local + local) and a stable
//        counting sort of own routed rows -> contiguous per-destination
//        segments; all-to-all of per-(destination, local expert) counts;
//      - one D2H of the routing report;
//   2. host: emits Algorithm 1 for the LOCAL experts (hot = predicted among
//      local experts, colds in demand order), sizes the exchange;
//   3. dispatch: NCCL all-to-all-v of the routed bf16 rows, local stable sort
//      of the received rows by local expert, expert FFNs (tcgen05),
//   4. return: gather to receive order, all-to-all-v back, weighted combine.
// The exchanges go through an Exchange backend:
//   * NcclExchange    one process per GPU (torchrun), NCCL all-reduce and
//                     grouped ncclSend/ncclRecv for the all-to-all-v. NCCL
//                     is resolved at run time (dlopen libnccl.so.2, the
//                     instance torch has loaded when present) so the library
//                     does not pin an NCCL build.
//   * LoopbackExchange G engines of ONE process on one device, each driven by
//                     its own host thread: every collective is a host
//                     rendezvous (publish buffers + a ready event), device
//                     copies pulled from the peers' buffers on the caller's
//                     stream after waiting on their events, and a second
//                     rendezvous so no rank reuses a buffer a peer is still
//                     reading. It runs the exact G>1 code path (relabel,
//                     counts exchange, dispatch, return, integer
//                     all-reduces, cross-rank demand) where only one GPU
//                     exists.
//   * SelfExchange    G = 1: device copies.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>

#include "engine.hpp"
#include "klotski/engine.h"
#include "klotski/kernels.h"

namespace klotski {

using namespace moesim;

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw moesim::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
void kl_check_impl(int rc, const char* what) {
    if (rc != 0) throw moesim::DeviceError(std::string(what) + ": " + kl_error_string(rc));
}
#define kl_check(rc, what) (++launches_, kl_check_impl((rc), (what)))

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
    static NcclApi api;
    static std::mutex mu;  // engines may be created from several host threads
    std::lock_guard<std::mutex> lk(mu);
    if (api.lib != nullptr) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) throw moesim::DeviceError("engine EP: libnccl.so.2 not found");
    auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (p == nullptr) throw moesim::DeviceError(std::string("engine EP: NCCL symbol missing: ") + n);
        return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.lib = h;
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw moesim::DeviceError(std::string(what) + ": " + nccl_api().error_string(r));
}

int hex_val(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    throw ConfigError("engine EP: bad nccl_id hex");
}

}  // namespace

// ---- exchange backends ----------------------------------------------------
struct Engine::Exchange {
    virtual ~Exchange() = default;
    // In-place integer sum over ranks (int32 or int64 elements).
    virtual void all_reduce_sum(void* buf, int64_t n, bool i64, cudaStream_t st) = 0;
    // Byte segments per peer: send[soff[r], +slen[r]) goes to rank r, which
    // receives it at recv[roff[me], +rlen[me]).
    virtual void all_to_all_v(const char* send, const std::vector<int64_t>& soff, const std::vector<int64_t>& slen,
                              char* recv, const std::vector<int64_t>& roff, const std::vector<int64_t>& rlen,
                              cudaStream_t st) = 0;
};

namespace {

struct SelfExchange final : Engine::Exchange {
    void all_reduce_sum(void*, int64_t, bool, cudaStream_t) override {}
    void all_to_all_v(const char* send, const std::vector<int64_t>& soff, const std::vector<int64_t>& slen, char* recv,
                      const std::vector<int64_t>& roff, const std::vector<int64_t>& rlen, cudaStream_t st) override {
        if (slen[0] != rlen[0]) throw AccountingError("engine EP: self exchange size mismatch");
        if (slen[0] > 0)
            cuda_check(cudaMemcpyAsync(recv + roff[0], send + soff[0], static_cast<size_t>(slen[0]),
                                       cudaMemcpyDeviceToDevice, st), "self exchange");
    }
};

struct NcclExchange final : Engine::Exchange {
    ncclComm_t comm = nullptr;
    int G = 1;
    NcclExchange(int world, int rank, const std::string& hex) : G(world) {
        NcclApi& api = nccl_api();
        ncclUniqueId id;
        if (hex.size() != 2 * sizeof(id.internal)) throw ConfigError("engine EP: nccl_id must be 256 hex chars");
        for (size_t i = 0; i < sizeof(id.internal); ++i)
            id.internal[i] = static_cast<char>(hex_val(hex[2 * i]) * 16 + hex_val(hex[2 * i + 1]));
        nccl_check(api.comm_init_rank(&comm, world, id, rank), "ncclCommInitRank");
    }
    ~NcclExchange() override {
        if (comm != nullptr) nccl_api().comm_destroy(comm);
    }
    void all_reduce_sum(void* buf, int64_t n, bool i64, cudaStream_t st) override {
        nccl_check(nccl_api().all_reduce(buf, buf, static_cast<size_t>(n), i64 ? ncclInt64 : ncclInt32, ncclSum, comm, st),
                   "ncclAllReduce");
    }
    void all_to_all_v(const char* send, const std::vector<int64_t>& soff, const std::vector<int64_t>& slen, char* recv,
                      const std::vector<int64_t>& roff, const std::vector<int64_t>& rlen, cudaStream_t st) override {
        NcclApi& api = nccl_api();
        nccl_check(api.group_start(), "ncclGroupStart");
        for (int r = 0; r < G; ++r) {
            if (slen[r] > 0) nccl_check(api.send(send + soff[r], slen[r], ncclChar, r, comm, st), "ncclSend");
            if (rlen[r] > 0) nccl_check(api.recv(recv + roff[r], rlen[r], ncclChar, r, comm, st), "ncclRecv");
        }
        nccl_check(api.group_end(), "ncclGroupEnd");
    }
};

// Rendezvous point of one loopback group (process-global, by name).
struct LoopbackHub {
    struct Pub {
        const char* ptr = nullptr;
        cudaEvent_t ev = nullptr;
        std::vector<int64_t> off, len;
    };
    explicit LoopbackHub(int g) : G(g), pub(g), done(g), joined(g, 0) {}
    const int G;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool broken = false;
    std::vector<Pub> pub;
    std::vector<cudaEvent_t> done;
    std::vector<char> joined;

    // All G ranks arrive before any leaves (generation-counted, reusable).
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) throw moesim::DeviceError("engine EP loopback: a peer left the group");
        const uint64_t gen = generation;
        if (++arrived == G) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        cv.wait(lk, [&] { return generation != gen || broken; });
        if (broken) throw moesim::DeviceError("engine EP loopback: a peer left the group");
    }
    void abandon() {
        std::lock_guard<std::mutex> lk(mu);
        broken = true;
        cv.notify_all();
    }
};

std::mutex g_hubs_mu;
std::map<std::string, std::weak_ptr<LoopbackHub>> g_hubs;

std::shared_ptr<LoopbackHub> join_hub(const std::string& name, int G, int rank) {
    std::lock_guard<std::mutex> lk(g_hubs_mu);
    std::shared_ptr<LoopbackHub> h = g_hubs[name].lock();
    if (!h) {
        h = std::make_shared<LoopbackHub>(G);
        g_hubs[name] = h;
    }
    if (h->G != G) throw ConfigError("engine EP loopback: group '" + name + "' has a different world size");
    if (h->joined[rank]) throw ConfigError("engine EP loopback: rank joined group '" + name + "' twice");
    h->joined[rank] = 1;
    return h;
}

struct LoopbackExchange final : Engine::Exchange {
    std::shared_ptr<LoopbackHub> hub;
    int G, me;
    cudaEvent_t ready = nullptr, copied = nullptr;
    int64_t* stage;        // [G][n] int64 staging for the all-reduce
    int64_t* launches;
    LoopbackExchange(const std::string& group, int world, int rank, int64_t* stage_buf, int64_t* launch_counter)
        : hub(join_hub(group, world, rank)), G(world), me(rank), stage(stage_buf), launches(launch_counter) {
        cuda_check(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming), "event");
    }
    ~LoopbackExchange() override {
        hub->abandon();  // a peer blocked in a rendezvous fails instead of hanging
        cudaEventDestroy(ready);
        cudaEventDestroy(copied);
    }
    // Phase 1: publish (ptr, segments) + ready event; rendezvous.
    void publish(const char* ptr, const std::vector<int64_t>& off, const std::vector<int64_t>& len, cudaStream_t st) {
        cuda_check(cudaEventRecord(ready, st), "ready");
        {
            std::lock_guard<std::mutex> lk(hub->mu);
            hub->pub[me] = {ptr, ready, off, len};
        }
        hub->barrier();
    }
    // Phase 3: record this rank's copies, rendezvous, then wait for every
    // peer's copies out of our buffers before the stream may reuse them.
    void complete(cudaStream_t st) {
        cuda_check(cudaEventRecord(copied, st), "copied");
        {
            std::lock_guard<std::mutex> lk(hub->mu);
            hub->done[me] = copied;
        }
        hub->barrier();
        for (int s = 0; s < G; ++s)
            if (s != me) cuda_check(cudaStreamWaitEvent(st, hub->done[s], 0), "wait peer copies");
    }
    void all_reduce_sum(void* buf, int64_t n, bool i64, cudaStream_t st) override {
        const int64_t esz = i64 ? 8 : 4;
        const int64_t bytes = n * esz;
        publish(static_cast<const char*>(buf), {0}, {bytes}, st);
        char* stg = reinterpret_cast<char*>(stage);
        for (int s = 0; s < G; ++s) {
            const LoopbackHub::Pub& p = hub->pub[s];
            if (s != me) cuda_check(cudaStreamWaitEvent(st, p.ev, 0), "wait peer");
            cuda_check(cudaMemcpyAsync(stg + s * bytes, p.ptr, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, st),
                       "all-reduce gather");
        }
        complete(st);
        // Rank-order sum of the G gathered rows (exact integers).
        if (!i64) {
            ++*launches;
            kl_check_impl(kl_sum_rows_i32(reinterpret_cast<const int32_t*>(stg), G, static_cast<int>(n),
                                          static_cast<int32_t*>(buf), st), "all-reduce sum");
        } else {
            cuda_check(cudaMemcpyAsync(buf, stg, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, st), "sum init");
            for (int s = 1; s < G; ++s) {
                ++*launches;
                kl_check_impl(kl_add_i64(static_cast<int64_t*>(buf), stage + s * n, n, st), "all-reduce sum");
            }
        }
    }
    void all_to_all_v(const char* send, const std::vector<int64_t>& soff, const std::vector<int64_t>& slen, char* recv,
                      const std::vector<int64_t>& roff, const std::vector<int64_t>& rlen, cudaStream_t st) override {
        publish(send, soff, slen, st);
        for (int s = 0; s < G; ++s) {
            const LoopbackHub::Pub& p = hub->pub[s];
            if (p.len[me] != rlen[s]) throw AccountingError("engine EP loopback: all-to-all size mismatch");
            if (rlen[s] == 0) continue;
            if (s != me) cuda_check(cudaStreamWaitEvent(st, p.ev, 0), "wait peer");
            cuda_check(cudaMemcpyAsync(recv + roff[s], p.ptr + p.off[me], static_cast<size_t>(rlen[s]),
                                       cudaMemcpyDeviceToDevice, st), "all-to-all copy");
        }
        complete(st);
    }
};

}  // namespace

void Engine::ep_init() {
    if (!ep_) return;
    if (G_ == 1)
        xch_ = new SelfExchange;
    else if (cfg_.ep_backend == "loopback")
        xch_ = new LoopbackExchange(cfg_.ep_group, G_, rank_, xstage_, &launches_);
    else
        xch_ = new NcclExchange(G_, rank_, cfg_.ep_nccl_id);
}

void Engine::ep_shutdown() {
    delete xch_;
    xch_ = nullptr;
}

// Last gate of the block, on the compute stream (see the file header, step 1).
void Engine::ep_after_gates(int step, int layer) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int n = plan_.n_batches, E = D_.E;
    const int64_t T = static_cast<int64_t>(n) * tokens_per_batch(step);
    int32_t* cur = idx_[idx_cur_];
    int32_t* prev = idx_[idx_cur_ ^ 1];
    kl_check(kl_sum_rows_i32(report_, n, E, hist_all_, cs), "hist sum");
    if (G_ > 1) xch_->all_reduce_sum(hist_all_, E, false, cs);
    int64_t* scores = reinterpret_cast<int64_t*>(report_ + 2LL * n * E + 16 - ((2LL * n * E) % 16));
    int64_t* marg_copy = scores + E;
    if (layer + 1 < D_.L) {
        const int64_t cells = layer == 0 ? E : static_cast<int64_t>(E) * E;
        cuda_check(cudaMemsetAsync(delta_, 0, cells * 8, cs), "memset delta");
        if (layer == 0)
            kl_check(kl_coact_update(nullptr, cur, T, D_.k, E, 0, nullptr, delta_, cs), "coact");
        else
            kl_check(kl_coact_update(prev, cur, T, D_.k, E, layer, delta_ - static_cast<int64_t>(layer - 1) * E * E,
                                     nullptr, cs),
                     "coact");
        if (G_ > 1) xch_->all_reduce_sum(delta_, cells, true, cs);
        kl_check(kl_add_i64(layer == 0 ? marginal_ : table_ + static_cast<int64_t>(layer - 1) * E * E, delta_, cells, cs),
                 "apply coact");
        kl_check(kl_predict_scores(hist_all_, table_, E, layer + 1, scores, cs), "predict");
    }
    // Own routed rows grouped by destination rank, then local expert.
    kl_check(kl_map_ids(cur, T * D_.k, label_map_, lbl_, cs), "relabel");
    // y_ret_ doubles as the send buffer (dispatch completes before return).
    shared_experts(layer, T, 0);  // replicated with the router: every rank on its own tokens
    kl_check(kl_permute(lbl_, T, D_.k, E, x2_, D_.d, send_counts_, offsets_, pos_, row_token_, y_ret_, perm_ws_, cs),
             "permute (dispatch order)");
    launches_ += kl_permute_launches(T * D_.k) - 1;
    // Per-(destination, local expert) counts exchange.
    {
        std::vector<int64_t> off(G_), len(G_, static_cast<int64_t>(El_) * 4);
        for (int r = 0; r < G_; ++r) off[r] = static_cast<int64_t>(r) * El_ * 4;
        xch_->all_to_all_v(reinterpret_cast<const char*>(send_counts_), off, len, reinterpret_cast<char*>(recv_counts_),
                           off, len, cs);
    }
    cuda_check(cudaMemcpyAsync(marg_copy, marginal_, E * 8, cudaMemcpyDeviceToDevice, cs), "marginal");
    // recv_counts and hist_all follow the report block in the same D2H.
    const size_t head = reinterpret_cast<char*>(marg_copy + E) - reinterpret_cast<char*>(report_);
    cuda_check(cudaMemcpyAsync(host_report_, report_, head, cudaMemcpyDeviceToHost, cs), "d2h report");
    cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(host_report_) + head, recv_counts_,
                               static_cast<size_t>(G_) * El_ * 4, cudaMemcpyDeviceToHost, cs), "d2h recv counts");
    if (cfg_.record_trace)
        cuda_check(cudaMemcpyAsync(host_idx_, cur, T * D_.k * 4, cudaMemcpyDeviceToHost, cs), "d2h idx");
    idx_cur_ ^= 1;
}

detail::BlockRouting Engine::ep_read_routing(int step, int layer) {
    const std::int32_t last_gate = next_exec_ - 1;
    cuda_check(cudaEventSynchronize(op_end_[last_gate]), "routing sync");
    const int n = plan_.n_batches, E = D_.E;
    const int32_t* hist = host_report_;
    const int32_t* first = host_report_ + static_cast<int64_t>(n) * E;
    const int64_t* scores = reinterpret_cast<const int64_t*>(host_report_ + 2LL * n * E + 16 - ((2LL * n * E) % 16));
    host_scores_.assign(scores, scores + E);
    host_marginal_.assign(scores + E, scores + 2 * E);
    const int32_t* rc = reinterpret_cast<const int32_t*>(scores + 2 * E);

    // Own per-global-expert counts -> per-destination send segments.
    std::vector<int64_t> own(E, 0);
    for (int b = 0; b < n; ++b)
        for (int e = 0; e < E; ++e) own[e] += hist[b * E + e];
    send_cnt_.assign(G_, 0);
    for (int e = 0; e < E; ++e) send_cnt_[e % G_] += own[e];
    send_off_.assign(G_ + 1, 0);
    for (int r = 0; r < G_; ++r) send_off_[r + 1] = send_off_[r] + send_cnt_[r];
    r_send_ = send_off_[G_];
    // Received rows: source-major, then local expert.
    recv_cnt_.assign(G_, 0);
    std::vector<int64_t> m_local(El_, 0);
    for (int s = 0; s < G_; ++s)
        for (int j = 0; j < El_; ++j) {
            recv_cnt_[s] += rc[s * El_ + j];
            m_local[j] += rc[s * El_ + j];
        }
    recv_off_.assign(G_ + 1, 0);
    for (int s = 0; s < G_; ++s) recv_off_[s + 1] = recv_off_[s] + recv_cnt_[s];
    r_recv_ = recv_off_[G_];
    for (int j = 0; j < El_; ++j) ep_max_local_rows_ = std::max(ep_max_local_rows_, m_local[j]);
    if (r_recv_ > r_recv_max_) throw AccountingError("engine EP: received rows exceed the exchange buffers");
    int64_t w = 0;
    for (int s = 0; s < G_; ++s)
        for (int j = 0; j < El_; ++j)
            for (int32_t c = 0; c < rc[s * El_ + j]; ++c) host_recv_ids_[w++] = j;

    // Algorithm-1 routing in the local view: local expert j = global j*G+rank.
    detail::BlockRouting r;
    r.group_hist = m_local;
    r.demand.resize(n);
    r.batch_hist.assign(n, std::vector<int64_t>(El_, 0));
    std::vector<char> demanded(El_, 0);
    for (int b = 0; b < n; ++b) {
        std::vector<std::pair<int32_t, int>> firsts;
        for (int j = 0; j < El_; ++j) {
            const int e = j * G_ + rank_;
            r.batch_hist[b][j] = hist[b * E + e];
            if (hist[b * E + e] > 0) firsts.emplace_back(first[b * E + e], j);
        }
        std::sort(firsts.begin(), firsts.end());
        for (const auto& [f, j] : firsts) {
            r.demand[b].push_back(j);
            demanded[j] = 1;
        }
    }
    for (int j = 0; j < El_; ++j)  // demanded only by other ranks' tokens
        if (m_local[j] > 0 && !demanded[j]) r.demand[n - 1].push_back(j);
    row_offset_.assign(El_, 0);
    for (int j = 1; j < El_; ++j) row_offset_[j] = row_offset_[j - 1] + m_local[j - 1];
    block_rows_ = r_recv_;
    batch_prefix_.assign(n, std::vector<int64_t>(El_, 0));
    if (cfg_.record_trace) {
        const size_t off = recorded_.offset(step, layer, 0, 0);
        const int64_t cnt = static_cast<int64_t>(n) * tokens_per_batch(step) * D_.k;
        for (int64_t i = 0; i < cnt; ++i) recorded_.sel[off + i] = static_cast<uint16_t>(host_idx_[i]);
    }
    return r;
}

// Row segments (offsets / counts in rows) -> byte segments for the backend.
void Engine::exchange_rows(const char* send, const std::vector<int64_t>& soff, const std::vector<int64_t>& scnt,
                           char* recv, const std::vector<int64_t>& roff, const std::vector<int64_t>& rcnt,
                           int64_t row_bytes, cudaStream_t st) {
    std::vector<int64_t> so(G_), sl(G_), ro(G_), rl(G_);
    for (int r = 0; r < G_; ++r) {
        so[r] = soff[r] * row_bytes;
        sl[r] = scnt[r] * row_bytes;
        ro[r] = roff[r] * row_bytes;
        rl[r] = rcnt[r] * row_bytes;
    }
    xch_->all_to_all_v(send, so, sl, recv, ro, rl, st);
}

void Engine::ep_dispatch() {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int64_t row_bytes = static_cast<int64_t>(D_.d) * 2;
    if (r_recv_ > 0)
        cuda_check(cudaMemcpyAsync(recv_ids_, host_recv_ids_, r_recv_ * 4, cudaMemcpyHostToDevice, cs), "h2d recv ids");
    exchange_rows(reinterpret_cast<const char*>(y_ret_), send_off_, send_cnt_, reinterpret_cast<char*>(recv_x_),
                  recv_off_, recv_cnt_, row_bytes, cs);
    kl_check(kl_permute(recv_ids_, r_recv_, 1, El_, recv_x_, D_.d, counts2_, offsets2_, pos2_, row_token2_, xp_,
                        perm_ws_, cs),
             "permute (local experts)");
    launches_ += kl_permute_launches(r_recv_) - 1;
}

void Engine::ep_return(int64_t T) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int64_t row_bytes = static_cast<int64_t>(D_.d) * 2;
    if (r_recv_ > 0) kl_check(kl_embed(pos2_, y_, r_recv_, D_.d, y_back_, cs), "gather to receive order");
    exchange_rows(reinterpret_cast<const char*>(y_back_), recv_off_, recv_cnt_, reinterpret_cast<char*>(y_ret_),
                  send_off_, send_cnt_, row_bytes, cs);
    kl_check(kl_combine(y_ret_, pos_, weight_, h_, T, D_.k, D_.d, h_, cs), "combine");
    if (cfg_.record_hidden) {
        std::vector<uint16_t> dump(static_cast<size_t>(T) * D_.d);
        cuda_check(cudaMemcpyAsync(dump.data(), h_, dump.size() * 2, cudaMemcpyDeviceToHost, cs), "dump");
        cuda_check(cudaStreamSynchronize(cs), "dump sync");
        hidden_dumps_.push_back(std::move(dump));
    }
}

}  // namespace klotski

extern "C" int kl_ep_unique_id(char* hex_out) {
    try {
        klotski::NcclApi& api = klotski::nccl_api();
        ncclUniqueId id;
        if (api.get_unique_id(&id) != ncclSuccess) return 1;
        static const char* digits = "0123456789abcdef";
        for (size_t i = 0; i < sizeof(id.internal); ++i) {
            const unsigned char c = static_cast<unsigned char>(id.internal[i]);
            hex_out[2 * i] = digits[c >> 4];
            hex_out[2 * i + 1] = digits[c & 15];
        }
        hex_out[2 * sizeof(id.internal)] = '\0';
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
