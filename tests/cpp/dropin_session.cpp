// dropin_session.cpp -- the reference's own model with the WG-KV hot path
// swapped for the B200 C-ABI, checked with the reference's engine KATs.
//
// TEST INFRASTRUCTURE (built into oracle/_ref/ by oracle/Makefile; links the
// reference library compiled from /root/reference and libwgkv_b200.so).
//
// B200Session is what a maintainer gets after applying INTEGRATION.md's patch
// to wgkv::Session: the ToyModel forward of Session::prefill /
// Session::decode_step (engine.cpp:153-341) -- embedding, RMSNorm, the Q/K/V
// projections, Wo and the GELU MLP stay on the host in fp64 exactly as the
// reference computes them -- while everything between the projections and Wo
// (RoPE, gate_forward_batch / gate_forward, binarize, build_vs_mask,
// attn_vertical_slash, prefill_populate, local_write + promote, gather,
// attn_ragged, select_topk_pages) runs on the GPU through wgkv_b200.hpp.
//
// The KATs restate tests/test_engine.cpp of the reference (file:line cited
// per case) against B200Session, with the reference's 1e-8 / 1e-10
// tolerances replaced by the fp32 device path's (kTolF32, stated per check)
// and, for the bf16 Llama-geometry case, the bf16 one.  Bits are compared
// with the reference's own Session: equal except tokens whose reference gate
// lies within 1e-6 of tau (reported).
//
// Usage: dropin_session  -> prints one line per KAT, exit code 0 iff all pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "wgkv/engine.hpp"
#include "wgkv/oracle.hpp"
#include "wgkv_b200.hpp"

using namespace wgkv;

namespace {

int g_fail = 0;
void report(const std::string& name, bool ok, const std::string& detail) {
    std::printf("KAT %-58s %s  %s\n", name.c_str(), ok ? "PASS" : "FAIL", detail.c_str());
    if (!ok) ++g_fail;
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// device buffer of raw bytes
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    void ensure(size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFree(p);
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
        n = bytes;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

uint16_t to_bf16(float f) {  // round to nearest even
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
float from_bf16(uint16_t h) {
    uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

b200::Policy to_b200(const PolicyConfig& p) {
    b200::Policy o;
    switch (p.kind) {
        case PolicyKind::full: o.kind = b200::PolicyKind::full; break;
        case PolicyKind::wgkv: o.kind = b200::PolicyKind::wgkv; break;
        case PolicyKind::local_sink: o.kind = b200::PolicyKind::local_sink; break;
        case PolicyKind::static_heads: o.kind = b200::PolicyKind::static_heads; break;
        case PolicyKind::wgkv_plus_topk: o.kind = b200::PolicyKind::wgkv_plus_topk; break;
    }
    o.window = p.window;
    o.sink = p.sink;
    o.retrieval_bitmap = p.retrieval_bitmap;
    o.topk_budget = p.topk_budget;
    o.forced.mode = static_cast<b200::ForcedAdmission::Mode>(static_cast<int>(p.forced.mode));
    o.forced.keep_every = p.forced.keep_every;
    o.forced.phase = p.forced.phase;
    o.forced.fraction = p.forced.fraction;
    return o;
}

wgkv_config make_config(const ToyModel& m, const GateBank& gates, const PolicyConfig& pol, long max_tokens,
                        int dtype) {
    wgkv_config c{};
    c.layers = m.cfg.layers;
    c.q_heads = m.cfg.q_heads;
    c.kv_heads = m.cfg.kv_heads;
    c.head_dim = m.cfg.head_dim;
    c.hidden = gates.hidden();
    c.window = pol.window;
    c.tau = pol.threshold.tau;
    c.rope_base = m.cfg.rope_base;
    c.page_size = 16;  // engine.cpp:102
    c.max_seqs = 1;
    c.max_tokens = max_tokens;
    c.max_prefill_tokens = max_tokens;
    c.dtype = dtype;
    c.topk_budget = pol.kind == PolicyKind::wgkv_plus_topk ? pol.topk_budget : 0;
    return c;
}

// ---------------------------------------------------------------------------
// Session with the hot path on the B200 (engine.cpp:153-341 host parts kept)
// ---------------------------------------------------------------------------
class B200Session {
public:
    B200Session(const ToyModel& model, const GateBank& gates, const PolicyConfig& policy, long max_total_tokens,
                int dtype = WGKV_F32)
        : model_(model),
          policy_(policy),
          bpol_(to_b200(policy)),
          dtype_(dtype),
          dev_(make_config(model, gates, policy, max_total_tokens, dtype)),
          trace_(model.cfg.layers, model.cfg.kv_heads) {
        if (policy.kind == PolicyKind::static_heads &&
            policy.retrieval_bitmap.size() != static_cast<size_t>(model.cfg.layers) * model.cfg.kv_heads)
            throw std::invalid_argument("Session: retrieval_bitmap must have layers * kv_heads entries");
        // GateBank -> the C-ABI's flat blocks W1 | b1 | w2 | b2 (gating.hpp:41-68)
        std::vector<double> bank;
        for (int l = 0; l < gates.layers(); ++l)
            for (int h = 0; h < gates.heads(); ++h) {
                const GateParams& p = gates.at(l, h);
                bank.insert(bank.end(), p.w1.data.begin(), p.w1.data.end());
                bank.insert(bank.end(), p.b1.begin(), p.b1.end());
                bank.insert(bank.end(), p.w2.begin(), p.w2.end());
                bank.push_back(p.b2);
            }
        dev_.set_gates(bank.data(), gates.layers(), gates.heads());
    }

    Matrix prefill(std::span<const int> tokens) {
        const auto& cfg = model_.cfg;
        const long T = static_cast<long>(tokens.size());
        if (T == 0) throw std::invalid_argument("Session::prefill: empty prompt");
        prompt_len_ = T;
        const int d = cfg.head_dim, dim = cfg.model_dim(), Hq = cfg.q_heads, Hkv = cfg.kv_heads;
        Matrix x(T, dim);
        for (long t = 0; t < T; ++t) {
            const int id = tokens[static_cast<size_t>(t)];
            if (id < 0 || id >= cfg.vocab) throw std::invalid_argument("Session::prefill: unknown token id");
            const auto e = model_.embed.row(id);
            std::copy(e.begin(), e.end(), x.row(t).begin());
        }
        std::vector<double> q(T * Hq * d), k(T * Hkv * d), v(T * Hkv * d), out(T * Hq * d);
        std::vector<float> g(Hkv * T);
        std::vector<uint8_t> bits(Hkv * T);
        for (int l = 0; l < cfg.layers; ++l) {
            const auto& w = model_.layers[static_cast<size_t>(l)];
            Matrix a(T, dim);
            for (long t = 0; t < T; ++t) {
                const auto n = rmsnorm(x.row(t), cfg.rms_eps);
                std::copy(n.begin(), n.end(), a.row(t).begin());
            }
            // projections (engine.cpp:191-198, 226-228), pre-RoPE; layout [T][heads][d]
            for (long t = 0; t < T; ++t) {
                for (int h = 0; h < Hkv; ++h)
                    for (int r = 0; r < d; ++r) {
                        k[(t * Hkv + h) * d + r] = dot(w.wk.row(h * d + r), a.row(t));
                        v[(t * Hkv + h) * d + r] = dot(w.wv.row(h * d + r), a.row(t));
                    }
                for (int p = 0; p < Hq; ++p)
                    for (int r = 0; r < d; ++r) q[(t * Hq + p) * d + r] = dot(w.wq.row(p * d + r), a.row(t));
            }
            const float* forced = upload_forced(l, 0, T);
            // the hot path: K1 (RoPE + gate + binarize) -> K2 (prefill_populate) -> K3 (VS attention)
            dev_.prefill_layer(l, 0, 1, T, upload(q, dq_), upload(k, dk_), upload(v, dv_), out_buf(T * Hq * d),
                               forced, (float*)dbuf(dg_, g.size() * 4), (uint8_t*)dbuf(dbits_, bits.size()));
            download(out, T * Hq * d);
            cuda_check(cudaMemcpy(g.data(), dg_.p, g.size() * 4, cudaMemcpyDeviceToHost), "g");
            cuda_check(cudaMemcpy(bits.data(), dbits_.p, bits.size(), cudaMemcpyDeviceToHost), "bits");
            for (int h = 0; h < Hkv; ++h)
                for (long t = 0; t < T; ++t) trace_.record(l, h, g[h * T + t], bits[h * T + t] != 0);
            // Wo + MLP (engine.cpp:243-250); concat = out [T][Hq*d]
            for (long t = 0; t < T; ++t) {
                auto xr = x.row(t);
                std::span<const double> concat(out.data() + t * Hq * d, static_cast<size_t>(Hq * d));
                for (int r = 0; r < dim; ++r) xr[r] += dot(w.wo.row(r), concat);
                const auto b = rmsnorm(xr, cfg.rms_eps);
                std::vector<double> hm(static_cast<size_t>(cfg.mlp_hidden));
                for (int r = 0; r < cfg.mlp_hidden; ++r) hm[static_cast<size_t>(r)] = gelu(dot(w.w_mlp1.row(r), b));
                for (int r = 0; r < dim; ++r) xr[r] += dot(w.w_mlp2.row(r), hm);
            }
        }
        dev_.sync();
        Matrix hidden(T, dim);
        for (long t = 0; t < T; ++t) {
            const auto n = rmsnorm(x.row(t), cfg.rms_eps);
            std::copy(n.begin(), n.end(), hidden.row(t).begin());
        }
        next_pos_ = T;
        return hidden;
    }

    std::vector<double> decode_step(int token) {
        const auto& cfg = model_.cfg;
        if (token < 0 || token >= cfg.vocab) throw std::invalid_argument("Session::decode_step: unknown token id");
        const long pos = next_pos_++;
        const int d = cfg.head_dim, dim = cfg.model_dim(), Hq = cfg.q_heads, Hkv = cfg.kv_heads;
        const auto e = model_.embed.row(token);
        std::vector<double> x(e.begin(), e.end());
        std::vector<double> q(Hq * d), k(Hkv * d), v(Hkv * d), concat(Hq * d);
        std::vector<float> g(Hkv);
        std::vector<uint8_t> bits(Hkv), near(Hkv);
        std::vector<int32_t> ev(Hkv);
        for (int l = 0; l < cfg.layers; ++l) {
            const auto& w = model_.layers[static_cast<size_t>(l)];
            const auto a = rmsnorm(x, cfg.rms_eps);
            for (int h = 0; h < Hkv; ++h)
                for (int r = 0; r < d; ++r) {
                    k[h * d + r] = dot(w.wk.row(h * d + r), a);
                    v[h * d + r] = dot(w.wv.row(h * d + r), a);
                }
            for (int p = 0; p < Hq; ++p)
                for (int r = 0; r < d; ++r) q[p * d + r] = dot(w.wq.row(p * d + r), a);
            const float* forced = upload_forced(l, pos, 1);
            wgkv_decode_trace tr{(float*)dbuf(dg_, Hkv * 4), (uint8_t*)dbuf(dbits_, Hkv),
                                 (uint8_t*)dbuf(dnear_, Hkv), (int32_t*)dbuf(dev_ev_, Hkv * 4)};
            // the hot path: gate_forward + local_write (K4) and gather + attn_ragged (K5 / K6)
            dev_.decode_layer(l, 0, 1, upload(q, dq_), upload(k, dk_), upload(v, dv_), out_buf(Hq * d), forced, tr);
            download(concat, Hq * d);
            cuda_check(cudaMemcpy(g.data(), tr.g, Hkv * 4, cudaMemcpyDeviceToHost), "g");
            cuda_check(cudaMemcpy(bits.data(), tr.bits, Hkv, cudaMemcpyDeviceToHost), "bits");
            cuda_check(cudaMemcpy(near.data(), tr.near_tau, Hkv, cudaMemcpyDeviceToHost), "near");
            for (int h = 0; h < Hkv; ++h) {
                trace_.record(l, h, g[h], bits[h] != 0);
                near_tau_ += near[h];
            }
            for (int r = 0; r < dim; ++r) x[static_cast<size_t>(r)] += dot(w.wo.row(r), concat);
            const auto b = rmsnorm(x, cfg.rms_eps);
            std::vector<double> hm(static_cast<size_t>(cfg.mlp_hidden));
            for (int r = 0; r < cfg.mlp_hidden; ++r) hm[static_cast<size_t>(r)] = gelu(dot(w.w_mlp1.row(r), b));
            for (int r = 0; r < dim; ++r) x[static_cast<size_t>(r)] += dot(w.w_mlp2.row(r), hm);
        }
        dev_.sync();
        return logits_from_hidden_row(model_, rmsnorm(x, cfg.rms_eps));
    }

    const GateTrace& trace() const { return trace_; }
    long position() const { return next_pos_; }
    long near_tau() const { return near_tau_; }
    b200::Device::Gathered gather(int l, int h) { return dev_.gather(l, 0, h, model_.cfg.head_dim); }

private:
    // policy override of the MLP gate (engine.cpp:126-151) -> forced_g on the device
    const float* upload_forced(int layer, long pos0, long T) {
        std::vector<float> fg;
        if (!b200::policy_gates(bpol_, layer, 0, model_.cfg.kv_heads, model_.cfg.kv_heads, 1, pos0, T, prompt_len_,
                                fg))
            return nullptr;
        void* p = dbuf(dforced_, fg.size() * 4);
        cuda_check(cudaMemcpy(p, fg.data(), fg.size() * 4, cudaMemcpyHostToDevice), "forced");
        return static_cast<const float*>(p);
    }
    static void* dbuf(DevBuf& b, size_t bytes) {
        b.ensure(std::max<size_t>(bytes, 16));
        return b.p;
    }
    size_t esize() const { return dtype_ == WGKV_BF16 ? 2 : 4; }
    // fp64 host values -> device in the context's dtype
    const void* upload(const std::vector<double>& x, DevBuf& b) {
        void* p = dbuf(b, x.size() * esize());
        if (dtype_ == WGKV_BF16) {
            std::vector<uint16_t> h(x.size());
            for (size_t i = 0; i < x.size(); ++i) h[i] = to_bf16(static_cast<float>(x[i]));
            cuda_check(cudaMemcpy(p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
        } else {
            std::vector<float> h(x.begin(), x.end());
            cuda_check(cudaMemcpy(p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload");
        }
        return p;
    }
    void* out_buf(size_t n) { return dbuf(dout_, n * esize()); }
    void download(std::vector<double>& y, size_t n) {
        if (dtype_ == WGKV_BF16) {
            std::vector<uint16_t> h(n);
            cuda_check(cudaMemcpy(h.data(), dout_.p, n * 2, cudaMemcpyDeviceToHost), "download");
            for (size_t i = 0; i < n; ++i) y[i] = from_bf16(h[i]);
        } else {
            std::vector<float> h(n);
            cuda_check(cudaMemcpy(h.data(), dout_.p, n * 4, cudaMemcpyDeviceToHost), "download");
            for (size_t i = 0; i < n; ++i) y[i] = h[i];
        }
    }

    const ToyModel& model_;
    PolicyConfig policy_;
    b200::Policy bpol_;
    int dtype_;
    b200::Device dev_;
    GateTrace trace_;
    long prompt_len_ = 0, next_pos_ = 0, near_tau_ = 0;
    DevBuf dq_, dk_, dv_, dout_, dg_, dbits_, dnear_, dev_ev_, dforced_;
};

// generate() (engine.cpp) on the B200 session: prefill + greedy argmax steps
std::vector<int> b200_generate(const ToyModel& model, const GateBank& gates, std::span<const int> prompt, long steps,
                               const PolicyConfig& policy) {
    B200Session s(model, gates, policy, static_cast<long>(prompt.size()) + steps);
    std::vector<int> ids(prompt.begin(), prompt.end());
    const Matrix hidden = s.prefill(prompt);
    std::vector<double> logits = logits_from_hidden_row(model, hidden.row(hidden.rows - 1));
    for (long i = 0; i < steps; ++i) {
        const int next = argmax_token(logits);
        ids.push_back(next);
        if (i + 1 < steps) logits = s.decode_step(next);
    }
    return ids;
}

// ---- the reference test file's helpers (test_engine.cpp:14-47), restated --
ModelConfig small_config() {
    ModelConfig cfg;
    cfg.layers = 2;
    cfg.q_heads = 4;
    cfg.kv_heads = 4;
    cfg.head_dim = 16;
    cfg.mlp_hidden = 64;
    cfg.vocab = 64;
    return cfg;
}
std::vector<int> random_prompt(long n, int vocab, uint64_t seed) {
    Rng rng(seed);
    std::vector<int> prompt(static_cast<size_t>(n));
    for (auto& t : prompt) t = static_cast<int>(rng.uniform_int(0, vocab));
    return prompt;
}
GateBank spread_gates(const ModelConfig& cfg, uint64_t seed) {
    return GateBank::random_init(cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.head_dim, seed, 0.5, -2.5);
}
GateBank saturated_gates(const ModelConfig& cfg, uint64_t seed, double b2) {
    return GateBank::random_init(cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.head_dim, seed, 0.02, b2);
}
double max_abs_diff(const Matrix& a, const Matrix& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::abs(a.data[i] - b.data[i]));
    return m;
}
double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}
double max_abs(const std::vector<double>& a) {
    double m = 0.0;
    for (double x : a) m = std::max(m, std::abs(x));
    return m;
}
char buf[256];
const char* fmt(const char* f, double a, double b = 0, double c = 0) {
    std::snprintf(buf, sizeof buf, f, a, b, c);
    return buf;
}

// fp32 device path: inputs rounded to fp32 (2^-24), fp32 attention; hidden
// states are O(1) after RMSNorm, logits O(10)
constexpr double kTolF32 = 1e-4;

// bits of our trace vs the reference Session's trace: equal except where the
// reference gate is within 1e-6 of tau (north_star); returns mismatches outside
long trace_mismatch(const GateTrace& ours, const GateTrace& ref, double tau, long* near_out) {
    long bad = 0, near = 0;
    for (int l = 0; l < ref.layers; ++l)
        for (int h = 0; h < ref.heads; ++h) {
            const auto& rb = ref.bits[l][h];
            const auto& ob = ours.bits[l][h];
            if (rb.size() != ob.size()) return 1 << 30;
            for (size_t j = 0; j < rb.size(); ++j) {
                const bool nt = std::abs(ref.gates[l][h][j] - tau) < 1e-6;
                near += nt;
                if (rb[j] != ob[j] && !nt) ++bad;
            }
        }
    if (near_out) *near_out = near;
    return bad;
}

// ---- KATs ---------------------------------------------------------------------
void kat_full_equals_teacher() {  // test_engine.cpp:49-66
    const auto cfg = small_config();
    const ToyModel model = ToyModel::random(cfg, 1);
    const GateBank gates = spread_gates(cfg, 2);
    const auto prompt = random_prompt(40, cfg.vocab, 3);
    PolicyConfig policy;
    policy.kind = PolicyKind::full;
    policy.window = 8;
    B200Session session(model, gates, policy, 40);
    const Matrix hidden = session.prefill(prompt);
    const double e = max_abs_diff(hidden, teacher_forward(model, prompt));
    bool resident = true;
    for (int l = 0; l < cfg.layers; ++l)
        for (int h = 0; h < cfg.kv_heads; ++h) {
            const auto g = session.gather(l, h);
            resident &= g.local_len + g.global_len == 40;
        }
    report("policy=full equals the dense teacher, caches every token", e < kTolF32 && resident,
           fmt("max|hidden - teacher| %.2e (tol %.0e)", e, kTolF32));
}

void kat_saturated_and_zeroed() {  // test_engine.cpp:68-105
    const auto cfg = small_config();
    const ToyModel model = ToyModel::random(cfg, 11);
    const auto prompt = random_prompt(48, cfg.vocab, 12);
    PolicyConfig wgkv_policy;
    wgkv_policy.kind = PolicyKind::wgkv;
    wgkv_policy.window = 8;
    PolicyConfig full_policy = wgkv_policy;
    full_policy.kind = PolicyKind::full;
    const GateBank sat = saturated_gates(cfg, 13, 20.0);
    const auto a = b200_generate(model, sat, prompt, 16, wgkv_policy);
    const auto b = b200_generate(model, sat, prompt, 16, full_policy);
    const auto r = generate(model, sat, prompt, 16, wgkv_policy).first;
    B200Session sa(model, sat, wgkv_policy, 48), sb(model, sat, full_policy, 48);
    const double e = max_abs_diff(sa.prefill(prompt), sb.prefill(prompt));
    report("saturated gates reproduce full attention", a == b && a == r && e < kTolF32,
           fmt("ids equal (and = reference generate), max|wgkv - full| %.2e", e));
    const GateBank zeroed = saturated_gates(cfg, 13, -20.0);
    PolicyConfig sliding = wgkv_policy;
    sliding.kind = PolicyKind::local_sink;
    sliding.sink = 0;
    const auto c = b200_generate(model, zeroed, prompt, 16, wgkv_policy);
    const auto d = b200_generate(model, zeroed, prompt, 16, sliding);
    const auto rz = generate(model, zeroed, prompt, 16, wgkv_policy).first;
    report("zeroed gates reproduce the sliding window", c == d && c == rz, "generated ids equal");
}

// test_engine.cpp:107-152 (and :154-178 with kv_heads = 2 / window 4)
void kat_masked_oracle(const char* name, const ModelConfig& cfg, uint64_t mseed, const GateBank& gates, long T,
                       long steps, long window, int dtype, double tol, uint64_t pseed) {
    const ToyModel model = ToyModel::random(cfg, mseed);
    const auto prompt = random_prompt(T, cfg.vocab, pseed);
    const double tau = 0.1;
    PolicyConfig policy;
    policy.kind = PolicyKind::wgkv;
    policy.window = window;
    policy.threshold = Threshold{tau};
    B200Session session(model, gates, policy, T + steps, dtype);
    Session ref(model, gates, policy, T + steps);  // the reference's own Session, for the bits
    const Matrix hidden = session.prefill(prompt);
    const Matrix ref_sess_hidden = ref.prefill(prompt);
    MaskedOracle oracle(model, window);
    const Matrix ref_hidden = oracle.prefill(prompt, session.trace());
    double eh = max_abs_diff(hidden, ref_hidden), el = 0.0, lmax = 0.0;
    (void)ref_sess_hidden;
    bool audit = true;
    std::vector<double> logits = logits_from_hidden_row(model, hidden.row(hidden.rows - 1));
    for (long step = 0; step < steps; ++step) {
        const int next = argmax_token(logits);
        logits = session.decode_step(next);
        ref.decode_step(next);
        const auto ref_logits = oracle.decode_step(next, session.trace());
        el = std::max(el, max_abs_diff(logits, ref_logits));
        lmax = std::max(lmax, max_abs(ref_logits));
        // exhaustive promotion audit after every step
        const long t_now = session.position() - 1;
        for (int l = 0; l < cfg.layers; ++l)
            for (int h = 0; h < cfg.kv_heads; ++h) {
                const auto kv = session.gather(l, h);
                const auto& b_hist = session.trace().bits[l][h];
                std::set<long> global_set(kv.global_pos.begin(), kv.global_pos.end());
                for (long j = 0; j <= t_now; ++j) {
                    const bool expected = j <= t_now - window && b_hist[static_cast<size_t>(j)] != 0;
                    audit &= global_set.count(j) == (expected ? 1u : 0u);
                }
                std::vector<long> expect_local;
                for (long j = std::max<long>(0, t_now - window + 1); j <= t_now; ++j) expect_local.push_back(j);
                audit &= kv.local_pos == expect_local;
            }
    }
    // bits vs the reference's own Session (fp32 inputs only: bf16-rounded keys
    // legitimately move gate scores, MaskedOracle then replays our bits)
    long near = 0;
    const long bad = dtype == WGKV_F32 ? trace_mismatch(session.trace(), ref.trace(), tau, &near) : 0;
    const double rel_l = el / std::max(lmax, 1e-30);
    const bool ok = eh < tol && rel_l < tol && audit && bad == 0;
    std::snprintf(buf, sizeof buf,
                  "hidden %.2e, logits rel %.2e (tol %.0e); audit %s; bits vs reference Session: %ld off, "
                  "%ld near-tau",
                  eh, rel_l, tol, audit ? "ok" : "FAILED", bad, near);
    report(name, ok, buf);
}

void kat_local_sink_accounting() {  // test_engine.cpp:196-213
    const auto cfg = small_config();
    const ToyModel model = ToyModel::random(cfg, 51);
    const GateBank gates = spread_gates(cfg, 52);
    const auto prompt = random_prompt(1000, cfg.vocab, 53);
    PolicyConfig policy;
    policy.kind = PolicyKind::local_sink;
    policy.window = 256;
    policy.sink = 128;
    B200Session session(model, gates, policy, 1000);
    session.prefill(prompt);
    bool ok = true;
    for (int l = 0; l < cfg.layers; ++l)
        for (int h = 0; h < cfg.kv_heads; ++h) {
            const auto g = session.gather(l, h);
            ok &= g.local_len == 256 && g.global_len == 128;
        }
    report("local_sink accounting at the reference operating point", ok, "local 256 / global 128 per head");
}

void kat_static_heads() {  // test_engine.cpp:241-286
    const auto cfg = small_config();
    const ToyModel model = ToyModel::random(cfg, 71);
    const GateBank gates = spread_gates(cfg, 72);
    const auto prompt = random_prompt(40, cfg.vocab, 73);
    const long window = 8;
    const size_t n_heads = static_cast<size_t>(cfg.layers) * cfg.kv_heads;
    PolicyConfig retrieval;
    retrieval.kind = PolicyKind::static_heads;
    retrieval.window = window;
    retrieval.retrieval_bitmap.assign(n_heads, 1);
    PolicyConfig full_policy;
    full_policy.kind = PolicyKind::full;
    full_policy.window = window;
    const bool ab = b200_generate(model, gates, prompt, 12, retrieval) == b200_generate(model, gates, prompt, 12,
                                                                                         full_policy);
    PolicyConfig streaming = retrieval;
    streaming.retrieval_bitmap.assign(n_heads, 0);
    PolicyConfig sliding;
    sliding.kind = PolicyKind::local_sink;
    sliding.window = window;
    sliding.sink = 0;
    const bool cd = b200_generate(model, gates, prompt, 12, streaming) == b200_generate(model, gates, prompt, 12,
                                                                                        sliding);
    PolicyConfig mixed = retrieval;
    for (size_t i = 0; i < n_heads; ++i) mixed.retrieval_bitmap[i] = i % 2 == 0 ? 1 : 0;
    B200Session session(model, gates, mixed, 40);
    session.prefill(prompt);
    bool resid = true;
    size_t idx = 0;
    for (int l = 0; l < cfg.layers; ++l)
        for (int h = 0; h < cfg.kv_heads; ++h, ++idx) {
            const auto g = session.gather(l, h);
            resid &= g.global_len == (mixed.retrieval_bitmap[idx] ? 40 - window : 0) && g.local_len == window;
        }
    PolicyConfig bad = mixed;
    bad.retrieval_bitmap.pop_back();
    bool threw = false;
    try {
        B200Session s(model, gates, bad, 40);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    report("static_heads policy behaviors", ab && cd && resid && threw,
           "retrieval==full, streaming==sliding, mixed residency, bitmap length rejected");
}

void kat_lifecycle_errors() {  // test_engine.cpp (Session lifecycle) / kvstore "out of pages"
    const auto cfg = small_config();
    const ToyModel model = ToyModel::random(cfg, 91);
    const GateBank gates = spread_gates(cfg, 92);
    PolicyConfig policy;
    policy.window = 8;
    bool ok = true;
    {
        B200Session s(model, gates, policy, 16);
        try {
            s.prefill(std::vector<int>{});
            ok = false;
        } catch (const std::invalid_argument&) {
        }
        try {
            s.prefill(std::vector<int>{1, 2, 99});
            ok = false;
        } catch (const std::invalid_argument&) {
        }
    }
    policy.threshold = Threshold{1.5};
    try {
        B200Session s(model, gates, policy, 16);
        ok = false;
    } catch (const std::invalid_argument&) {
    }
    report("lifecycle: empty prompt, unknown token, tau outside (0,1)", ok, "std::invalid_argument as the reference");
}

}  // namespace

int main() {
    try {
        kat_full_equals_teacher();
        kat_saturated_and_zeroed();
        {
            const auto cfg = small_config();
            kat_masked_oracle("wgkv prefill+decode = MaskedOracle, per-step promotion audit", cfg, 21,
                              spread_gates(cfg, 22), 48, 24, 8, WGKV_F32, kTolF32, 23);
        }
        {
            ModelConfig cfg = small_config();
            cfg.kv_heads = 2;
            kat_masked_oracle("grouped-query attention matches the oracle too", cfg, 31,
                              GateBank::random_init(cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.head_dim, 32, 0.5,
                                                    -2.5),
                              32, 8, 4, WGKV_F32, kTolF32, 33);
        }
        kat_local_sink_accounting();
        kat_static_heads();
        kat_lifecycle_errors();
        {
            // Llama-3.1-8B head geometry (d = 128, GQA 4) through the bf16 Blackwell
            // kernels (K1 tcgen05, K3 tcgen05, K5 mma.sync): bf16 tolerance 1e-2
            ModelConfig cfg;
            cfg.layers = 2;
            cfg.q_heads = 8;
            cfg.kv_heads = 2;
            cfg.head_dim = 128;
            cfg.mlp_hidden = 256;
            cfg.vocab = 64;
            cfg.rope_base = 500000.0;
            kat_masked_oracle("Llama head geometry (d=128, GQA 4), bf16 tcgen05/mma.sync path", cfg, 101,
                              GateBank::random_init(cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.head_dim, 102, 0.1,
                                                    -1.5),
                              300, 20, 64, WGKV_BF16, 2e-2, 103);
        }
    } catch (const std::exception& e) {
        std::printf("KAT harness error: %s\n", e.what());
        return 2;
    }
    std::printf("%s: %d failed\n", g_fail ? "FAIL" : "ALL PASS", g_fail);
    return g_fail ? 1 : 0;
}
