// ref_shim.cpp -- extern "C" face over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources straight from /root/reference/proj/src (never
// copied into this repo) into oracle/_ref/libwgkv_ref.so.  Uses:
//   * tests/test_oracle_vs_ref.py: the C restatement (wgkv_oracle.c) must be
//     bitwise equal to these calls on the same inputs;
//   * tests/golden/make_golden.py: golden vectors produced by the reference;
//   * bench.py --impl reference / cpu_baseline: the reference's own CPU path
//     (gate_forward_batch + build_vs_mask + attn_vertical_slash +
//     prefill_populate, then local_write + gather + attn_ragged per decode
//     step) timed on the host, parallel over heads with wgkv::parallel_for
//     exactly as Session does (engine.cpp:188-257, 291-327).
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "wgkv/attention.hpp"
#include "wgkv/engine.hpp"
#include "wgkv/gating.hpp"
#include "wgkv/kvstore.hpp"
#include "wgkv/numerics.hpp"

using namespace wgkv;

namespace {

int status_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::logic_error&) {
        return 3;
    } catch (const std::runtime_error& r) {
        return std::strncmp(r.what(), "out of pages", 12) == 0 ? 2 : 4;
    } catch (...) {
        return 4;
    }
}

Matrix to_matrix(const double* p, long rows, long cols) {
    Matrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data.data(), p, sizeof(double) * rows * cols);
    return m;
}

GateParams params_from_block(const double* blk, int d, int hidden) {
    GateParams p;
    p.w1 = to_matrix(blk, hidden, 2 * d);
    const double* b1 = blk + static_cast<long>(hidden) * 2 * d;
    p.b1.assign(b1, b1 + hidden);
    p.w2.assign(b1 + hidden, b1 + 2 * hidden);
    p.b2 = b1[2 * hidden];
    return p;
}

// Per-layer hot-path state for one sequence: pool + one HeadCache per
// (layer, kv head), as Session owns them (engine.hpp:106-107).
struct RefSession {
    int layers, q_heads, kv_heads, d, hidden;
    long window, topk;
    double tau, rope_base;
    std::vector<GateParams> bank;
    KvPool pool;
    std::vector<HeadCache> caches;
    RefSession(int L, int hq, int hkv, int d_, int hid, long W, double tau_, double base, int ps, long cap, long topk_,
               const double* gate_bank)
        : layers(L), q_heads(hq), kv_heads(hkv), d(d_), hidden(hid), window(W), topk(topk_), tau(tau_),
          rope_base(base), pool(ps, d_, cap) {
        const long blen = static_cast<long>(hid) * 2 * d_ + 2L * hid + 1;
        if (gate_bank)
            for (long b = 0; b < static_cast<long>(L) * hkv; ++b)
                bank.push_back(params_from_block(gate_bank + b * blen, d_, hid));
        for (int l = 0; l < L; ++l)
            for (int h = 0; h < hkv; ++h) caches.emplace_back(l, h, W);
    }
    HeadCache& at(int l, int h) { return caches[static_cast<size_t>(l) * kv_heads + h]; }
};

}  // namespace

extern "C" {

int wr_thread_budget() { return thread_budget(); }

void wr_gaussian_fill(uint64_t seed, double scale, double* out, long n) {
    Rng rng(seed);
    for (long i = 0; i < n; ++i) out[i] = scale * rng.gaussian();
}

void wr_uniform_fill(uint64_t seed, double* out, long n) {
    Rng rng(seed);
    for (long i = 0; i < n; ++i) out[i] = rng.uniform();
}

int wr_rope(double* k, int d, long pos, double base, double sign) {
    try {
        std::span<double> s(k, static_cast<size_t>(d));
        if (sign > 0)
            apply_rope_inplace(s, pos, RopeConfig{d, base});
        else
            apply_rope_inverse_inplace(s, pos, RopeConfig{d, base});
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

int wr_gate_random_init(int L, int H, int d, int hidden, uint64_t seed, double w_std, double b2, double* out) {
    try {
        const GateBank bank = GateBank::random_init(L, H, d, hidden, seed, w_std, b2);
        long o = 0;
        for (int l = 0; l < L; ++l)
            for (int h = 0; h < H; ++h) {
                const GateParams& p = bank.at(l, h);
                for (double x : p.w1.data) out[o++] = x;
                for (double x : p.b1) out[o++] = x;
                for (double x : p.w2) out[o++] = x;
                out[o++] = p.b2;
            }
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

int wr_gate_save(const char* path, int L, int H, int d, int hidden, const double* bank) {
    try {
        GateBank b(L, H, d, hidden);
        const long blen = static_cast<long>(hidden) * 2 * d + 2L * hidden + 1;
        for (int l = 0; l < L; ++l)
            for (int h = 0; h < H; ++h) b.at(l, h) = params_from_block(bank + (l * H + h) * blen, d, hidden);
        b.save(path);
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

int wr_gate_forward_batch(const double* blk, int d, int hidden, const double* k_pre, const double* k_post, long t,
                          double* g_out) {
    try {
        const auto g = gate_forward_batch(params_from_block(blk, d, hidden), to_matrix(k_pre, t, d),
                                          to_matrix(k_post, t, d));
        std::memcpy(g_out, g.data(), sizeof(double) * t);
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

int wr_binarize(const double* g, long n, double tau, uint8_t* bits) {
    try {
        const auto b = binarize(std::span<const double>(g, static_cast<size_t>(n)), Threshold{tau});
        std::memcpy(bits, b.data(), static_cast<size_t>(n));
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

int wr_attn_vertical_slash(const double* q, long tq, const double* k, const double* v, long tk, int d, double scale,
                           long causal_offset, long window, const uint8_t* admitted, double* out, uint64_t* evals) {
    try {
        const Matrix qm = to_matrix(q, tq, d), km = to_matrix(k, tk, d), vm = to_matrix(v, tk, d);
        VsMask mask{window, std::vector<uint8_t>(admitted, admitted + tk)};
        OpCounter c;
        const Matrix o = attn_vertical_slash({qm, km, vm, scale, causal_offset}, mask, &c);
        std::memcpy(out, o.data.data(), sizeof(double) * tq * d);
        if (evals) *evals += c.score_evals;
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

uint64_t wr_vs_pair_count(long window, const uint8_t* admitted, long nq, long nk, long off) {
    VsMask mask{window, std::vector<uint8_t>(admitted, admitted + nk)};
    return vs_mask_pair_count(mask, nq, nk, off);
}

int wr_attn_ragged(const double* q, const double* gk, const double* gv, long g_rows, const double* lk, const double* lv,
                   long l_rows, int d, double scale, double* out, uint64_t* evals) {
    try {
        OpCounter c;
        const auto o = attn_ragged(std::span<const double>(q, static_cast<size_t>(d)), to_matrix(gk, g_rows, d),
                                   to_matrix(gv, g_rows, d), to_matrix(lk, l_rows, d), to_matrix(lv, l_rows, d),
                                   scale, &c);
        std::memcpy(out, o.data(), sizeof(double) * d);
        if (evals) *evals += c.score_evals;
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// ---- path-level session over reference primitives ------------------------

void* wr_session_create(int L, int hq, int hkv, int d, int hidden, long W, double tau, double base, int ps, long cap,
                        long topk, const double* gate_bank) {
    try {
        return new RefSession(L, hq, hkv, d, hidden, W, tau, base, ps, cap, topk, gate_bank);
    } catch (...) {
        return nullptr;
    }
}

void wr_session_destroy(void* s) { delete static_cast<RefSession*>(s); }

// engine.cpp:188-257 with the projections removed; parallel over heads with
// the reference's own parallel_for (WGKV_THREADS) exactly as Session does.
int wr_session_prefill_layer(void* sp, int layer, const double* q_pre, const double* k_pre, const double* v, long t,
                             const double* forced_gates, double* out, double* g_out, uint8_t* bits_out,
                             uint64_t* evals) {
    auto& s = *static_cast<RefSession*>(sp);
    try {
        const int d = s.d, hkv = s.kv_heads, hq = s.q_heads, gsz = hq / hkv;
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        const RopeConfig rope{d, s.rope_base};
        std::vector<Matrix> k_post(static_cast<size_t>(hkv), Matrix(t, d)), vv(static_cast<size_t>(hkv), Matrix(t, d));
        std::vector<std::vector<double>> gates(static_cast<size_t>(hkv));
        std::vector<VsMask> masks(static_cast<size_t>(hkv));
        parallel_for(hkv, [&](long lo, long hi) {
            for (long h = lo; h < hi; ++h) {
                Matrix kp(t, d);
                for (long i = 0; i < t; ++i) {
                    std::memcpy(kp.row(i).data(), k_pre + (i * hkv + h) * d, sizeof(double) * d);
                    std::memcpy(k_post[h].row(i).data(), kp.row(i).data(), sizeof(double) * d);
                    apply_rope_inplace(k_post[h].row(i), i, rope);
                    std::memcpy(vv[h].row(i).data(), v + (i * hkv + h) * d, sizeof(double) * d);
                }
                if (forced_gates)
                    gates[h].assign(forced_gates + h * t, forced_gates + (h + 1) * t);
                else
                    gates[h] = gate_forward_batch(s.bank[static_cast<size_t>(layer) * hkv + h], kp, k_post[h]);
                masks[h] = build_vs_mask(gates[h], Threshold{s.tau}, s.window);
            }
        });
        std::vector<OpCounter> counters(static_cast<size_t>(hq));
        parallel_for(hq, [&](long lo, long hi) {
            for (long p = lo; p < hi; ++p) {
                const long h = p / gsz;
                Matrix q(t, d);
                for (long i = 0; i < t; ++i) {
                    std::memcpy(q.row(i).data(), q_pre + (i * hq + p) * d, sizeof(double) * d);
                    apply_rope_inplace(q.row(i), i, rope);
                }
                const Matrix o = attn_vertical_slash({q, k_post[h], vv[h], scale, 0}, masks[h], &counters[p]);
                for (long i = 0; i < t; ++i)
                    std::memcpy(out + (i * hq + p) * d, o.row(i).data(), sizeof(double) * d);
            }
        });
        for (int h = 0; h < hkv; ++h)
            s.at(layer, h).prefill_populate(s.pool, k_post[h], vv[h], gates[h], Threshold{s.tau}, 0);
        for (int h = 0; h < hkv; ++h) {
            if (g_out) std::memcpy(g_out + h * t, gates[h].data(), sizeof(double) * t);
            if (bits_out) std::memcpy(bits_out + h * t, masks[h].admitted.data(), static_cast<size_t>(t));
        }
        if (evals)
            for (const auto& c : counters) *evals += c.score_evals;
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// HeadCache::prefill_populate (kvstore.cpp:160-203) of every kv head of a
// layer with given gates, no attention: builds a long-context cache state for
// timing the reference's decode step (bench.py cpu_baseline).  k_pre, v
// [t][kv_heads][d]; gates [kv_heads][t].
int wr_session_populate_layer(void* sp, int layer, const double* k_pre, const double* v, const double* gates, long t) {
    auto& s = *static_cast<RefSession*>(sp);
    try {
        const int d = s.d, hkv = s.kv_heads;
        const RopeConfig rope{d, s.rope_base};
        std::vector<Matrix> k_post(static_cast<size_t>(hkv), Matrix(t, d)), vv(static_cast<size_t>(hkv), Matrix(t, d));
        parallel_for(hkv, [&](long lo, long hi) {
            for (long h = lo; h < hi; ++h)
                for (long i = 0; i < t; ++i) {
                    std::memcpy(k_post[h].row(i).data(), k_pre + (i * hkv + h) * d, sizeof(double) * d);
                    apply_rope_inplace(k_post[h].row(i), i, rope);
                    std::memcpy(vv[h].row(i).data(), v + (i * hkv + h) * d, sizeof(double) * d);
                }
        });
        for (int h = 0; h < hkv; ++h)
            s.at(layer, h).prefill_populate(s.pool, k_post[h], vv[h],
                                            std::vector<double>(gates + h * t, gates + (h + 1) * t),
                                            Threshold{s.tau}, 0);
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// engine.cpp:291-327 with the projections removed
int wr_session_decode_layer(void* sp, int layer, const double* q_pre, const double* k_pre, const double* v,
                            const double* forced_gates, double* out, double* g_out, int* events, uint64_t* evals) {
    auto& s = *static_cast<RefSession*>(sp);
    try {
        const int d = s.d, hkv = s.kv_heads, hq = s.q_heads, gsz = hq / hkv;
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        const RopeConfig rope{d, s.rope_base};
        const long pos = s.at(layer, 0).tokens_seen();
        std::vector<GatheredKv> gathered(static_cast<size_t>(hkv));
        OpCounter counter;
        for (int h = 0; h < hkv; ++h) {
            std::vector<double> kp(k_pre + h * d, k_pre + (h + 1) * d), vn(v + h * d, v + (h + 1) * d);
            const auto kr = apply_rope(kp, pos, rope);
            const double g = forced_gates ? forced_gates[h]
                                          : gate_forward(s.bank[static_cast<size_t>(layer) * hkv + h],
                                                         build_gate_feature(kp, kr));
            if (g_out) g_out[h] = g;
            const auto ev = s.at(layer, h).local_write(s.pool, kr, vn, g, Threshold{s.tau}, pos);
            if (events) events[h] = static_cast<int>(ev);
            gathered[h] = s.at(layer, h).gather(s.pool);
        }
        for (int p = 0; p < hq; ++p) {
            const int h = p / gsz;
            std::vector<double> q(q_pre + p * d, q_pre + (p + 1) * d);
            apply_rope_inplace(q, pos, rope);
            std::vector<double> o;
            if (s.topk > 0) {
                const auto sel = select_topk_pages(q, s.at(layer, h), s.pool, s.topk);
                o = attn_ragged(q, sel.k, sel.v, gathered[h].local_k, gathered[h].local_v, scale, &counter);
            } else {
                o = attn_ragged(q, gathered[h].global_k, gathered[h].global_v, gathered[h].local_k,
                                gathered[h].local_v, scale, &counter);
            }
            std::memcpy(out + p * d, o.data(), sizeof(double) * d);
        }
        if (evals) *evals += counter.score_evals;
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// Timed variant of wr_session_prefill_layer for the CPU baseline: the same
// three phases Session::prefill runs per layer (engine.cpp:188-257), each
// timed with a steady clock.  secs[0] = RoPE+gate_forward_batch+build_vs_mask
// (parallel over kv heads), secs[1] = RoPE(q)+attn_vertical_slash (parallel
// over q heads), secs[2] = prefill_populate (serial).  *pairs = score evals.
int wr_session_prefill_layer_timed(void* sp, int layer, const double* q_pre, const double* k_pre, const double* v,
                                   long t, double* secs, uint64_t* pairs) {
    auto& s = *static_cast<RefSession*>(sp);
    using clk = std::chrono::steady_clock;
    try {
        const int d = s.d, hkv = s.kv_heads, hq = s.q_heads, gsz = hq / hkv;
        const double scale = 1.0 / std::sqrt(static_cast<double>(d));
        const RopeConfig rope{d, s.rope_base};
        std::vector<Matrix> k_post(static_cast<size_t>(hkv), Matrix(t, d)), vv(static_cast<size_t>(hkv), Matrix(t, d));
        std::vector<std::vector<double>> gates(static_cast<size_t>(hkv));
        std::vector<VsMask> masks(static_cast<size_t>(hkv));
        auto t0 = clk::now();
        parallel_for(hkv, [&](long lo, long hi) {
            for (long h = lo; h < hi; ++h) {
                Matrix kp(t, d);
                for (long i = 0; i < t; ++i) {
                    std::memcpy(kp.row(i).data(), k_pre + (i * hkv + h) * d, sizeof(double) * d);
                    std::memcpy(k_post[h].row(i).data(), kp.row(i).data(), sizeof(double) * d);
                    apply_rope_inplace(k_post[h].row(i), i, rope);
                    std::memcpy(vv[h].row(i).data(), v + (i * hkv + h) * d, sizeof(double) * d);
                }
                gates[h] = gate_forward_batch(s.bank[static_cast<size_t>(layer) * hkv + h], kp, k_post[h]);
                masks[h] = build_vs_mask(gates[h], Threshold{s.tau}, s.window);
            }
        });
        auto t1 = clk::now();
        std::vector<OpCounter> counters(static_cast<size_t>(hq));
        parallel_for(hq, [&](long lo, long hi) {
            for (long p = lo; p < hi; ++p) {
                Matrix q(t, d);
                for (long i = 0; i < t; ++i) {
                    std::memcpy(q.row(i).data(), q_pre + (i * hq + p) * d, sizeof(double) * d);
                    apply_rope_inplace(q.row(i), i, rope);
                }
                const Matrix o = attn_vertical_slash({q, k_post[p / gsz], vv[p / gsz], scale, 0}, masks[p / gsz],
                                                     &counters[p]);
                (void)o;
            }
        });
        auto t2 = clk::now();
        for (int h = 0; h < hkv; ++h)
            s.at(layer, h).prefill_populate(s.pool, k_post[h], vv[h], gates[h], Threshold{s.tau}, 0);
        auto t3 = clk::now();
        secs[0] = std::chrono::duration<double>(t1 - t0).count();
        secs[1] = std::chrono::duration<double>(t2 - t1).count();
        secs[2] = std::chrono::duration<double>(t3 - t2).count();
        *pairs = 0;
        for (const auto& c : counters) *pairs += c.score_evals;
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// lens[0..3] = local_len, local_ptr, global_len, tokens_seen
int wr_session_head_state(void* sp, int layer, int h, long* lens) {
    auto& c = static_cast<RefSession*>(sp)->at(layer, h);
    lens[0] = c.local_len();
    lens[1] = c.local_ptr();
    lens[2] = c.global_len();
    lens[3] = c.tokens_seen();
    return 0;
}

int wr_session_gather(void* sp, int layer, int h, double* gk, double* gv, long* gpos, double* ggate, double* lk,
                      double* lv, long* lpos, double* lgate) {
    auto& s = *static_cast<RefSession*>(sp);
    const auto kv = s.at(layer, h).gather(s.pool);
    const size_t G = kv.global_pos.size(), L = kv.local_pos.size();
    if (gk) std::memcpy(gk, kv.global_k.data.data(), sizeof(double) * G * s.d);
    if (gv) std::memcpy(gv, kv.global_v.data.data(), sizeof(double) * G * s.d);
    if (gpos) std::memcpy(gpos, kv.global_pos.data(), sizeof(long) * G);
    if (ggate) std::memcpy(ggate, kv.global_gate.data(), sizeof(double) * G);
    if (lk) std::memcpy(lk, kv.local_k.data.data(), sizeof(double) * L * s.d);
    if (lv) std::memcpy(lv, kv.local_v.data.data(), sizeof(double) * L * s.d);
    if (lpos) std::memcpy(lpos, kv.local_pos.data(), sizeof(long) * L);
    if (lgate) std::memcpy(lgate, kv.local_gate.data(), sizeof(double) * L);
    return 0;
}

// cache_snapshot (kvstore.cpp:269-286) over the session's caches in Session
// order (layer-major, then kv head); *len = text length, copied (NUL
// terminated) when cap > len.
int wr_session_snapshot(void* sp, char* buf, long cap, long* len) {
    try {
        auto& s = *static_cast<RefSession*>(sp);
        const std::string t = cache_snapshot({s.caches.data(), s.caches.size()}, s.pool);
        *len = static_cast<long>(t.size());
        if (buf && cap > *len) {
            std::memcpy(buf, t.data(), t.size());
            buf[t.size()] = 0;
        }
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// cache_stats (kvstore.cpp:253-267) over every HeadCache of the session:
// out = {resident_entries, admitted_fraction, pages_allocated}
int wr_session_cache_stats(void* sp, double* out) {
    try {
        auto& s = *static_cast<RefSession*>(sp);
        const CacheStats st = cache_stats({s.caches.data(), s.caches.size()}, s.pool);
        out[0] = static_cast<double>(st.resident_entries);
        out[1] = st.admitted_fraction;
        out[2] = static_cast<double>(st.pages_allocated);
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

int wr_session_select_topk(void* sp, int layer, int h, const double* q, long budget, long* logical, long* n_sel) {
    auto& s = *static_cast<RefSession*>(sp);
    try {
        const auto sel = select_topk_pages(std::span<const double>(q, static_cast<size_t>(s.d)), s.at(layer, h),
                                           s.pool, budget);
        for (size_t i = 0; i < sel.logical_pages.size(); ++i) logical[i] = sel.logical_pages[i];
        *n_sel = static_cast<long>(sel.logical_pages.size());
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// Session::effective_gate as the reference applies it (engine.cpp:126-151):
// a real wgkv::Session over ToyModel::random with the given policy runs
// prefill(T tokens) + n_decode decode steps; the GateTrace it records
// (engine.cpp:214-217, 305) is copied out as out_g[L][H][T + n_decode].
// kind: 0 full, 1 wgkv, 2 local_sink, 3 static_heads, 4 wgkv_plus_topk
// (PolicyKind order, engine.hpp:17); fmode: 0 none, 1 stride, 2 recent_fraction.
int wr_policy_trace(int kind, long window, long sink, const uint8_t* bitmap, int fmode, long keep_every, long phase,
                    double fraction, int L, int H, long T, int n_decode, double* out_g) {
    try {
        ModelConfig mc;
        mc.layers = L;
        mc.q_heads = H;
        mc.kv_heads = H;
        mc.head_dim = 8;
        mc.mlp_hidden = 16;
        mc.vocab = 32;
        const ToyModel model = ToyModel::random(mc, 7);
        const GateBank gates = GateBank::random_init(L, H, mc.head_dim, mc.head_dim, 11, 0.5, 0.0);
        PolicyConfig pc;
        pc.kind = static_cast<PolicyKind>(kind);
        pc.window = window;
        pc.sink = sink;
        if (bitmap) pc.retrieval_bitmap.assign(bitmap, bitmap + static_cast<size_t>(L) * H);
        pc.forced.mode = static_cast<ForcedAdmission::Mode>(fmode);
        pc.forced.keep_every = keep_every;
        pc.forced.phase = phase;
        pc.forced.fraction = fraction;
        Session sess(model, gates, pc, T + n_decode);
        std::vector<int> tokens(static_cast<size_t>(T));
        for (long t = 0; t < T; ++t) tokens[static_cast<size_t>(t)] = static_cast<int>((t * 7 + 3) % mc.vocab);
        sess.prefill(tokens);
        for (int n = 0; n < n_decode; ++n) sess.decode_step((n * 5 + 1) % mc.vocab);
        const GateTrace& tr = sess.trace();
        for (int l = 0; l < L; ++l)
            for (int h = 0; h < H; ++h)
                for (long t = 0; t < T + n_decode; ++t)
                    out_g[(static_cast<size_t>(l) * H + h) * (T + n_decode) + t] =
                        tr.gates[static_cast<size_t>(l)][static_cast<size_t>(h)][static_cast<size_t>(t)];
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

}  // extern "C"
