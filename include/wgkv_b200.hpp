// wgkv_b200.hpp -- header-only C++ face of the C-ABI with the reference's
// names, argument meaning and exception classes (namespace wgkv::b200).
//
// A reference user replaces, per layer, the calls Session::prefill /
// Session::decode_step make (engine.cpp:188-257, 291-327):
//   gate_forward_batch + binarize      -> Device::gate_forward_batch   (K1)
//   HeadCache::prefill_populate        -> Device::prefill_populate     (K2)
//   build_vs_mask + attn_vertical_slash-> Device::attn_vertical_slash  (K3)
//   gate_forward + HeadCache::local_write -> Device::local_write       (K4)
//   HeadCache::gather + attn_ragged    -> Device::attn_ragged          (K5)
//   (select_topk_pages when topk_budget > 0)
// or the fused per-layer bodies Device::prefill_layer / decode_layer.
// Status codes map back to std::invalid_argument / std::runtime_error
// ("out of pages ...") / std::logic_error like the reference throws them
// (SURVEY.md §5).  All tensors are device pointers (see wgkv_b200.h).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "wgkv_b200.h"

namespace wgkv {
namespace b200 {

inline void throw_on(int status, const char* what) {
    if (status == WGKV_OK) return;
    const std::string msg = std::string(what) + ": " + wgkv_last_error();
    switch (status) {
        case WGKV_EINVAL: throw std::invalid_argument(msg);
        case WGKV_ESTATE: throw std::logic_error(msg);
        case WGKV_ENOPAGES:  // the reference's message starts with "out of pages"
            throw std::runtime_error(std::string(wgkv_last_error()));
        default: throw std::runtime_error(msg);
    }
}

class Device {
public:
    explicit Device(const wgkv_config& cfg) { throw_on(wgkv_ctx_create(&cfg, &ctx_), "Session::Session"); }
    ~Device() { wgkv_ctx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    void set_stream(void* cuda_stream) { throw_on(wgkv_set_stream(ctx_, cuda_stream), "set_stream"); }
    void sync() { throw_on(wgkv_sync(ctx_), "sync"); }
    // GateBank::load (gating.cpp:107-147)
    void load_gates(const std::string& path) { throw_on(wgkv_gate_load(ctx_, path.c_str()), "GateBank::load"); }
    void set_gates(const double* bank, int layers, int heads) {
        throw_on(wgkv_gate_set(ctx_, bank, layers, heads), "GateBank");
    }

    // gate_forward_batch + binarize (gating.cpp:173-190), RoPE fused
    void gate_forward_batch(int layer, int nseq, long T, long pos0, const void* k_pre, void* k_post, float* g,
                            uint8_t* bits) {
        throw_on(wgkv_gate_score(ctx_, layer, nseq, T, pos0, k_pre, nullptr, k_post, g, bits, nullptr, 0, nullptr),
                 "gate_forward_batch");
    }
    // HeadCache::prefill_populate (kvstore.cpp:160-203) for every kv head of the slots
    void prefill_populate(int layer, int seq0, int nseq, long T, const void* k_post, const void* v, const float* g,
                          const uint8_t* bits) {
        throw_on(wgkv_admit_prefill(ctx_, layer, seq0, nseq, T, k_post, v, g, bits), "prefill_populate");
    }
    // build_vs_mask + attn_vertical_slash (attention.cpp:116-153); q pre-RoPE
    void attn_vertical_slash(int layer, int seq0, int nseq, long T, const void* q, const void* k_post, const void* v,
                             const uint8_t* bits, void* out) {
        throw_on(wgkv_vs_prefill(ctx_, layer, seq0, nseq, T, q, k_post, v, bits, out), "attn_vertical_slash");
    }
    void prefill_layer(int layer, int seq0, int nseq, long T, const void* q, const void* k_pre, const void* v,
                       void* out, const float* forced_g = nullptr, float* g = nullptr, uint8_t* bits = nullptr) {
        throw_on(wgkv_prefill_layer(ctx_, layer, seq0, nseq, T, q, k_pre, v, forced_g, out, g, bits),
                 "Session::prefill");
    }
    // gate_forward + HeadCache::local_write with lazy promotion (kvstore.cpp:122-158)
    void local_write(int layer, int seq0, int nseq, const void* k_pre, const void* v, const float* forced_g = nullptr,
                     float* g = nullptr, int32_t* events = nullptr) {
        throw_on(wgkv_decode_step_kv(ctx_, layer, seq0, nseq, k_pre, v, forced_g, g, events), "local_write");
    }
    // HeadCache::gather + attn_ragged (kvstore.cpp:205-241, attention.cpp:155-180), in place
    void attn_ragged(int layer, int seq0, int nseq, const void* q, void* out) {
        throw_on(wgkv_decode_attn(ctx_, layer, seq0, nseq, q, out), "attn_ragged");
    }
    void decode_layer(int layer, int seq0, int nseq, const void* q, const void* k_pre, const void* v, void* out,
                      const float* forced_g = nullptr, float* g = nullptr, int32_t* events = nullptr) {
        throw_on(wgkv_decode_layer(ctx_, layer, seq0, nseq, q, k_pre, v, forced_g, out, g, events),
                 "Session::decode_step");
    }
    // decode_layer with the step's GateTrace (engine.cpp:300-305): g, g >= tau,
    // the near-tau flag and the ring victim's promotion event, device pointers
    void decode_layer(int layer, int seq0, int nseq, const void* q, const void* k_pre, const void* v, void* out,
                      const float* forced_g, const wgkv_decode_trace& trace) {
        throw_on(wgkv_decode_layer_traced(ctx_, layer, seq0, nseq, q, k_pre, v, forced_g, out, &trace),
                 "Session::decode_step");
    }
    // HeadCache accessors + gather (kvstore.hpp:120-127, kvstore.cpp:205-241) of one
    // (layer, seq, kv head), to host memory; with_kv = false copies positions and gates only
    struct Gathered {
        long local_len = 0, local_ptr = 0, global_len = 0, tokens_seen = 0, local_pages = 0, global_pages = 0;
        std::vector<long> global_pos, local_pos;
        std::vector<float> global_gate, local_gate;
        std::vector<float> global_k, global_v, local_k, local_v;  // [rows][d] when with_kv
    };
    Gathered gather(int layer, int seq, int kv_head, int head_dim, bool with_kv = false) {
        int64_t lens[6];
        throw_on(wgkv_cache_state(ctx_, layer, seq, kv_head, lens), "HeadCache::gather");
        Gathered g;
        g.local_len = lens[0], g.local_ptr = lens[1], g.global_len = lens[2], g.tokens_seen = lens[3];
        g.local_pages = lens[4], g.global_pages = lens[5];
        std::vector<int64_t> gp(g.global_len), lp(g.local_len);
        g.global_gate.resize(g.global_len);
        g.local_gate.resize(g.local_len);
        if (with_kv) {
            g.global_k.resize(g.global_len * head_dim), g.global_v.resize(g.global_len * head_dim);
            g.local_k.resize(g.local_len * head_dim), g.local_v.resize(g.local_len * head_dim);
        }
        throw_on(wgkv_cache_export(ctx_, layer, seq, kv_head, with_kv ? g.global_k.data() : nullptr,
                                   with_kv ? g.global_v.data() : nullptr, gp.data(), g.global_gate.data(),
                                   with_kv ? g.local_k.data() : nullptr, with_kv ? g.local_v.data() : nullptr,
                                   lp.data(), g.local_gate.data()),
                 "HeadCache::gather");
        g.global_pos.assign(gp.begin(), gp.end());
        g.local_pos.assign(lp.begin(), lp.end());
        return g;
    }
    // HeadCache::release (kvstore.cpp:243-251) for every head of the slots
    void release(int seq0, int nseq) { throw_on(wgkv_release(ctx_, seq0, nseq), "release"); }
    // cache_snapshot (kvstore.cpp:269-286) of one sequence slot (gate digits of the stored fp32 value)
    std::string cache_snapshot(int seq = 0) {
        size_t n = 0;
        throw_on(wgkv_cache_snapshot(ctx_, seq, nullptr, 0, &n), "cache_snapshot");
        std::string text(n + 1, '\0');
        throw_on(wgkv_cache_snapshot(ctx_, seq, text.data(), text.size(), &n), "cache_snapshot");
        text.resize(n);
        return text;
    }

    wgkv_ctx* handle() const { return ctx_; }

private:
    wgkv_ctx* ctx_ = nullptr;
};


// ---------------------------------------------------------------------------
// PolicyConfig / ForcedAdmission (engine.hpp:17-40) and Session::effective_gate
// (engine.cpp:126-151): the policy override of the MLP gate.  The device path
// takes it as the optional forced_g buffer of wgkv_gate_score /
// wgkv_prefill_layer / wgkv_decode_step_kv / wgkv_decode_layer (nullptr = the
// MLP decides); policy_gates() fills that buffer on the host.
// ---------------------------------------------------------------------------
enum class PolicyKind { full, wgkv, local_sink, static_heads, wgkv_plus_topk };

struct ForcedAdmission {
    enum class Mode { none, stride, recent_fraction };
    Mode mode = Mode::none;
    long keep_every = 4;     // stride: admit positions with pos % keep_every == phase
    long phase = 0;
    double fraction = 0.25;  // recent_fraction: admit the newest fraction of pre-window prompt positions
};

struct Policy {
    PolicyKind kind = PolicyKind::wgkv;
    long window = 256;
    long sink = 128;
    std::vector<uint8_t> retrieval_bitmap;  // static_heads: layers * kv_heads entries
    long topk_budget = 0;                   // wgkv_plus_topk (wgkv_config::topk_budget)
    ForcedAdmission forced;
};

// true when the gate MLP decides (engine.cpp:203): pass forced_g = nullptr
inline bool uses_mlp_gates(const Policy& p) {
    return (p.kind == PolicyKind::wgkv || p.kind == PolicyKind::wgkv_plus_topk) &&
           p.forced.mode == ForcedAdmission::Mode::none;
}

// effective gate of (layer, global kv head, position) when the MLP does not decide
inline double effective_gate(const Policy& p, int layer, int head, int kv_heads, long position, long prompt_len) {
    switch (p.kind) {
        case PolicyKind::full: return 1.0;
        case PolicyKind::local_sink: return position < p.sink ? 1.0 : 0.0;
        case PolicyKind::static_heads:
            return p.retrieval_bitmap.at(static_cast<size_t>(layer) * kv_heads + head) ? 1.0 : 0.0;
        case PolicyKind::wgkv:
        case PolicyKind::wgkv_plus_topk:
            switch (p.forced.mode) {
                case ForcedAdmission::Mode::none: break;
                case ForcedAdmission::Mode::stride:
                    return position % p.forced.keep_every == p.forced.phase ? 1.0 : 0.0;
                case ForcedAdmission::Mode::recent_fraction: {
                    const long pre_window = prompt_len - p.window > 0 ? prompt_len - p.window : 0;
                    const long cutoff = pre_window - static_cast<long>(std::llround(p.forced.fraction * pre_window));
                    return position >= cutoff ? 1.0 : 0.0;
                }
            }
    }
    throw std::logic_error("effective_gate: the gate MLP decides under this policy");
}

// forced_g for positions [pos0, pos0 + T) of nseq sequences and the local kv
// heads [kv_head_offset, kv_head_offset + kv_heads_local) of kv_heads_total:
// out = [nseq][kv_heads_local][T] (copy it to the device).  Returns false
// (and leaves out empty) when the MLP decides.
inline bool policy_gates(const Policy& p, int layer, int kv_head_offset, int kv_heads_local, int kv_heads_total,
                         int nseq, long pos0, long T, long prompt_len, std::vector<float>& out) {
    out.clear();
    if (uses_mlp_gates(p)) return false;
    out.resize(static_cast<size_t>(nseq) * kv_heads_local * T);
    for (int s = 0; s < nseq; ++s)
        for (int h = 0; h < kv_heads_local; ++h)
            for (long t = 0; t < T; ++t)
                out[(static_cast<size_t>(s) * kv_heads_local + h) * T + t] = static_cast<float>(
                    effective_gate(p, layer, kv_head_offset + h, kv_heads_total, pos0 + t, prompt_len));
    return true;
}

}  // namespace b200
}  // namespace wgkv
