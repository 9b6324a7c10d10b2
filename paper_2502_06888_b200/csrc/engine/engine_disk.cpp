// SPDX-License-Identifier: Apache-2.0
// Disk tier and the DRAM staging window.
//
// Reference semantics: plan_placement spills whole tensor classes of late
// layers to disk behind a window of cpu_window_L layers (placement.cpp:
// 156-218); window_advance stages layer (cur + L) mod n_layers and evicts cur
// at the end of every block (placement.cpp:245-255); the schedule carries
// these as window_stage ops on the cpu_stage stream, after every load of the
// evicted layer, and the loads of a disk layer depend on its latest stage op
// (schedule.cpp:374-426, 455-470).
//
// Here the disk is a real file: one region per layer holding that layer's
// disk-tier tensors in streamed format ([experts | gate | attention], only
// the parts whose tier is disk). A window_stage op frees the evicted layer's
// pinned window slot and reads the staged layer's region into a free slot
// with pread, from a host function enqueued on the cpu_stage CUDA stream
// (so its cross-stream dependencies are ordinary events, and the H2D loads
// of the staged layer wait on its end event). The file is unlinked right
// after creation; it disappears with the engine.
#include <fcntl.h>
#include <unistd.h>

#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "engine.hpp"

namespace klotski {

using namespace moesim;

byte_count Engine::disk_bytes(int layer) const {
    return plan_.placement.disk_bytes_of_layer(layer, spec_, cfg_.quant);
}

// Offset of a tensor class inside a layer's disk region.
byte_count Engine::disk_part_offset(int layer, TensorClass cls) const {
    const auto& pl = plan_.placement;
    byte_count off = 0;
    if (cls == TensorClass::expert) return off;
    if (pl.expert_tier[layer] == Tier::disk) off += expert_slot_bytes_ * El_;
    if (cls == TensorClass::gate) return off;
    if (pl.gate_tier[layer] == Tier::disk) off += spec_.gate_bytes;
    return off;  // attention
}

// A disk tensor is normally read from the window slot its layer was staged
// into. The reference schedule can also load a disk tensor of a layer that
// is not staged at that point: the next layer's attention is prefetched one
// block ahead, and its dependency on staged_latest_ is -1 (never staged) or
// a stage op of an earlier pass whose slot has since been evicted
// (stage_dep, schedule.cpp:146-153, with a window shorter than the prefetch
// distance).
// Those loads read the tensor straight from the file into the load stream's
// bounce buffer first (stream order keeps the buffer single-use).
const void* Engine::load_src(TensorClass cls, int layer, int e, cudaStream_t st) {
    const auto& pl = plan_.placement;
    const Tier t = cls == TensorClass::expert ? pl.expert_tier[layer]
                   : cls == TensorClass::gate ? pl.gate_tier[layer]
                                              : pl.attention_tier[layer];
    if (t != Tier::disk) {
        if (cls == TensorClass::expert) return host_expert_[static_cast<size_t>(layer) * El_ + e];
        return cls == TensorClass::gate ? host_gate_[layer] : host_attn_[layer];
    }
    const byte_count part = disk_part_offset(layer, cls) + (cls == TensorClass::expert ? expert_slot_bytes_ * e : 0);
    if (const int s = window_slot_of_[layer]; s >= 0) return window_slot_[s] + part;
    const byte_count bytes = cls == TensorClass::expert ? expert_slot_bytes_
                             : cls == TensorClass::gate ? spec_.gate_bytes
                                                        : attn_slot_bytes_;
    char* dst = bounce_[st == stream_of(StreamId::expert_load) ? 1 : 0];
    if (dst == nullptr || bytes > bounce_bytes_) throw AccountingError("engine: no bounce buffer for a direct disk read");
    enqueue_disk_read(dst, disk_off_[layer] + part, bytes, st);
    ++direct_reads_;
    direct_bytes_ += bytes;
    return dst;
}

void Engine::enqueue_disk_read(char* dst, int64_t off, int64_t bytes, cudaStream_t st) {
    stage_jobs_.push_back({this, dst, off, bytes});
    const cudaError_t e = cudaLaunchHostFunc(st, &Engine::stage_host_fn, &stage_jobs_.back());
    if (e != cudaSuccess) throw moesim::DeviceError(std::string("engine: disk read enqueue: ") + cudaGetErrorString(e));
}

void Engine::open_disk_store() {
    std::string dir = cfg_.disk_dir;
    if (dir.empty()) {
        const char* t = std::getenv("TMPDIR");
        dir = t != nullptr && *t != '\0' ? t : "/tmp";
    }
    std::string path = dir + "/klotski-disk-XXXXXX";
    std::vector<char> buf(path.begin(), path.end());
    buf.push_back('\0');
    disk_fd_ = ::mkstemp(buf.data());
    if (disk_fd_ < 0) throw moesim::DeviceError("engine: cannot create the disk store in " + dir + ": " + std::strerror(errno));
    ::unlink(buf.data());
    disk_off_.assign(D_.L, 0);
    int64_t off = 0;
    for (int l = 0; l < D_.L; ++l) {
        disk_off_[l] = off;
        off += disk_bytes(l);
    }
    disk_bytes_total_ = off;
    if (::ftruncate(disk_fd_, off) != 0)
        throw moesim::DeviceError(std::string("engine: cannot size the disk store: ") + std::strerror(errno));
}

// Host-function body: runs on the CUDA driver's callback thread, so no CUDA
// calls and no exceptions; a failure is recorded and raised at step end.
void Engine::stage_read(const StageJob& job) {
    char* dst = job.dst;
    int64_t left = job.bytes, off = job.off;
    while (left > 0) {
        const ssize_t r = ::pread(disk_fd_, dst, static_cast<size_t>(left), off);
        if (r <= 0) {
            stage_errno_.store(r == 0 ? EIO : errno);
            return;
        }
        dst += r;
        off += r;
        left -= r;
        disk_bytes_read_.fetch_add(r, std::memory_order_relaxed);
    }
}

void CUDART_CB Engine::stage_host_fn(void* p) {
    auto* job = static_cast<StageJob*>(p);
    job->eng->stage_read(*job);
}

}  // namespace klotski
