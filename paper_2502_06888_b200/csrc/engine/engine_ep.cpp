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
// NCCL is resolved at run time (dlopen libnccl.so.2, the instance torch has
// loaded when present) so the library does not pin an NCCL build.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
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
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void kl_check_impl(int rc, const char* what) {
    if (rc != 0) throw std::runtime_error(std::string(what) + ": " + kl_error_string(rc));
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
    if (api.lib != nullptr) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) throw std::runtime_error("engine EP: libnccl.so.2 not found");
    auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (p == nullptr) throw std::runtime_error(std::string("engine EP: NCCL symbol missing: ") + n);
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
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl_api().error_string(r));
}

int hex_val(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    throw ConfigError("engine EP: bad nccl_id hex");
}

}  // namespace

struct Engine::Nccl {
    ncclComm_t comm = nullptr;
};

void Engine::ep_init() {
    if (!ep_) return;
    nccl_ = new Nccl;
    if (G_ == 1) return;  // self exchange is a device copy; no communicator needed
    NcclApi& api = nccl_api();
    ncclUniqueId id;
    if (cfg_.ep_nccl_id.size() != 2 * sizeof(id.internal)) throw ConfigError("engine EP: nccl_id must be 256 hex chars");
    for (size_t i = 0; i < sizeof(id.internal); ++i)
        id.internal[i] = static_cast<char>(hex_val(cfg_.ep_nccl_id[2 * i]) * 16 + hex_val(cfg_.ep_nccl_id[2 * i + 1]));
    nccl_check(api.comm_init_rank(&nccl_->comm, G_, id, rank_), "ncclCommInitRank");
}

void Engine::ep_shutdown() {
    if (nccl_ == nullptr) return;
    if (nccl_->comm != nullptr) nccl_api().comm_destroy(nccl_->comm);
    delete nccl_;
    nccl_ = nullptr;
}

// Last gate of the block, on the compute stream (see the file header, step 1).
void Engine::ep_after_gates(int step, int layer) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int n = plan_.n_batches, E = D_.E;
    const int64_t T = static_cast<int64_t>(n) * tokens_per_batch(step);
    int32_t* cur = idx_[idx_cur_];
    int32_t* prev = idx_[idx_cur_ ^ 1];
    NcclApi* api = G_ > 1 ? &nccl_api() : nullptr;

    kl_check(kl_sum_rows_i32(report_, n, E, hist_all_, cs), "hist sum");
    if (api) nccl_check(api->all_reduce(hist_all_, hist_all_, E, ncclInt32, ncclSum, nccl_->comm, cs), "allreduce hist");
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
        if (api) nccl_check(api->all_reduce(delta_, delta_, cells, ncclInt64, ncclSum, nccl_->comm, cs), "allreduce coact");
        kl_check(kl_add_i64(layer == 0 ? marginal_ : table_ + static_cast<int64_t>(layer - 1) * E * E, delta_, cells, cs),
                 "apply coact");
        kl_check(kl_predict_scores(hist_all_, table_, E, layer + 1, scores, cs), "predict");
    }
    // Own routed rows grouped by destination rank, then local expert.
    kl_check(kl_map_ids(cur, T * D_.k, label_map_, lbl_, cs), "relabel");
    // y_ret_ doubles as the send buffer (dispatch completes before return).
    shared_experts(layer, T);  // replicated with the router: every rank on its own tokens
    kl_check(kl_permute(lbl_, T, D_.k, E, x2_, D_.d, send_counts_, offsets_, pos_, row_token_, y_ret_, perm_ws_, cs),
             "permute (dispatch order)");
    launches_ += 2;
    // Per-(destination, local expert) counts exchange.
    if (api) {
        nccl_check(api->group_start(), "group");
        for (int r = 0; r < G_; ++r) {
            nccl_check(api->send(send_counts_ + static_cast<int64_t>(r) * El_, El_, ncclInt32, r, nccl_->comm, cs), "send counts");
            nccl_check(api->recv(recv_counts_ + static_cast<int64_t>(r) * El_, El_, ncclInt32, r, nccl_->comm, cs), "recv counts");
        }
        nccl_check(api->group_end(), "group end");
    } else {
        cuda_check(cudaMemcpyAsync(recv_counts_, send_counts_, El_ * 4, cudaMemcpyDeviceToDevice, cs), "self counts");
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

void Engine::ep_dispatch() {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int64_t row_bytes = static_cast<int64_t>(D_.d) * 2;
    if (r_recv_ > 0)
        cuda_check(cudaMemcpyAsync(recv_ids_, host_recv_ids_, r_recv_ * 4, cudaMemcpyHostToDevice, cs), "h2d recv ids");
    if (G_ > 1) {
        NcclApi& api = nccl_api();
        nccl_check(api.group_start(), "group");
        for (int r = 0; r < G_; ++r) {
            if (send_cnt_[r] > 0)
                nccl_check(api.send(y_ret_ + send_off_[r] * D_.d, send_cnt_[r] * row_bytes, ncclChar, r, nccl_->comm, cs),
                           "dispatch send");
            if (recv_cnt_[r] > 0)
                nccl_check(api.recv(recv_x_ + recv_off_[r] * D_.d, recv_cnt_[r] * row_bytes, ncclChar, r, nccl_->comm, cs),
                           "dispatch recv");
        }
        nccl_check(api.group_end(), "group end");
    } else if (r_recv_ > 0) {
        cuda_check(cudaMemcpyAsync(recv_x_, y_ret_, r_recv_ * row_bytes, cudaMemcpyDeviceToDevice, cs), "self dispatch");
    }
    kl_check(kl_permute(recv_ids_, r_recv_, 1, El_, recv_x_, D_.d, counts2_, offsets2_, pos2_, row_token2_, xp_,
                        perm_ws_, cs),
             "permute (local experts)");
    launches_ += 2;
}

void Engine::ep_return(int64_t T) {
    cudaStream_t cs = stream_of(StreamId::compute);
    const int64_t row_bytes = static_cast<int64_t>(D_.d) * 2;
    if (r_recv_ > 0) kl_check(kl_embed(pos2_, y_, r_recv_, D_.d, y_back_, cs), "gather to receive order");
    if (G_ > 1) {
        NcclApi& api = nccl_api();
        nccl_check(api.group_start(), "group");
        for (int r = 0; r < G_; ++r) {
            if (recv_cnt_[r] > 0)
                nccl_check(api.send(y_back_ + recv_off_[r] * D_.d, recv_cnt_[r] * row_bytes, ncclChar, r, nccl_->comm, cs),
                           "return send");
            if (send_cnt_[r] > 0)
                nccl_check(api.recv(y_ret_ + send_off_[r] * D_.d, send_cnt_[r] * row_bytes, ncclChar, r, nccl_->comm, cs),
                           "return recv");
        }
        nccl_check(api.group_end(), "group end");
    } else if (r_recv_ > 0) {
        cuda_check(cudaMemcpyAsync(y_ret_, y_back_, r_recv_ * row_bytes, cudaMemcpyDeviceToDevice, cs), "self return");
    }
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
