// ref_glue.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/qcsim_oracle.c header).
//
// C-ABI shim over the reference's OWN codec/statevec/circuit translation
// units, compiled unmodified from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libqcsim_ref.so (-O3 -ffp-contract=off,
// SURVEY.md F7).  Used for: (1) generating tests/golden/ (the oracle's pin),
// (2) cross-checking the restatement, (3) the CPU baseline arm of bench.py
// (`--impl reference`): an engine loop over the reference's compress_plane /
// decompress_plane with a std::thread worker pool over slices.
// The reference has no engine source; the loop below follows
// the same pinned semantics as the oracle and the GPU engine.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "qcsim/circuit.hpp"
#include "qcsim/codec.hpp"
#include "qcsim/errors.hpp"
#include "qcsim/statevec.hpp"

#include "../include/qcsim_c.h"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

int classify(const std::exception &e) {
    if (dynamic_cast<const qcsim::CodecError *>(&e)) return QCSIM_CODEC;
    if (dynamic_cast<const qcsim::CapacityError *>(&e)) return QCSIM_CAPACITY;
    if (dynamic_cast<const qcsim::ParseError *>(&e)) return QCSIM_PARSE;
    if (dynamic_cast<const qcsim::NumericError *>(&e)) return QCSIM_NUMERIC;
    if (dynamic_cast<const std::invalid_argument *>(&e)) return QCSIM_INVALID_ARGUMENT;
    if (dynamic_cast<const std::bad_alloc *>(&e)) return QCSIM_NOMEM;
    return QCSIM_RUNTIME;
}

template <class F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return classify(e);
    }
}

qcsim::CodecConfig to_cfg(const qcsim_codec_config *c) {
    qcsim::CodecConfig cfg;
    cfg.mode = static_cast<qcsim::CodecMode>(c->mode);
    cfg.predictor = static_cast<qcsim::Predictor>(c->predictor);
    cfg.quant_code_bits = c->quant_code_bits;
    cfg.bound = c->bound;
    return cfg;
}

qcsim_action flatten(const qcsim::GateAction &ga) {
    qcsim_action a{};
    if (auto *d = std::get_if<qcsim::DiagonalOp>(&ga)) {
        a.kind = QCSIM_ACTION_DIAGONAL;
        a.mask = d->mask;
        a.factor[0] = d->factor.real();
        a.factor[1] = d->factor.imag();
    } else if (auto *b = std::get_if<qcsim::ButterflyOp>(&ga)) {
        a.kind = QCSIM_ACTION_BUTTERFLY;
        a.target = b->target;
        a.mask = b->control_mask;
        const qcsim::Amplitude u[4] = {b->u.u00, b->u.u01, b->u.u10, b->u.u11};
        for (int k = 0; k < 4; ++k) {
            a.u[2 * k] = u[k].real();
            a.u[2 * k + 1] = u[k].imag();
        }
    } else {
        auto &s = std::get<qcsim::SwapOp>(ga);
        a.kind = QCSIM_ACTION_SWAP;
        a.a = s.a;
        a.b = s.b;
    }
    return a;
}
} // namespace

EXPORT const char *ref_last_error() { return g_err.c_str(); }

EXPORT int ref_compress_plane(const double *v, uint64_t n, const qcsim_codec_config *c, uint8_t *out,
                              uint64_t cap, uint64_t *len, qcsim_codec_stats *st) {
    return guarded([&] {
        auto [blk, stats] = qcsim::compress_plane(std::span<const double>(v, n), to_cfg(c));
        auto bytes = blk.to_bytes();
        *len = bytes.size();
        if (out) {
            if (bytes.size() > cap) throw std::invalid_argument("output capacity too small");
            std::memcpy(out, bytes.data(), bytes.size());
        }
        if (st) {
            st->input_bytes = stats.input_bytes;
            st->output_bytes = stats.output_bytes;
            st->ratio = stats.ratio;
            st->outlier_fraction = stats.outlier_fraction;
        }
    });
}

EXPORT int ref_decompress_plane(const uint8_t *b, uint64_t len, double *out, uint64_t cap, uint64_t *n,
                                uint64_t *consumed) {
    return guarded([&] {
        size_t used = 0;
        auto blk = qcsim::CompressedBlock::from_bytes(std::span<const uint8_t>(b, len), &used);
        if (consumed) *consumed = used;
        auto vals = qcsim::decompress_plane(blk);
        *n = vals.size();
        if (out) {
            if (vals.size() > cap) throw std::invalid_argument("output capacity too small");
            std::memcpy(out, vals.data(), vals.size() * sizeof(double));
        }
    });
}

EXPORT double ref_planes_sq_norm(const double *re, const double *im, uint64_t n) {
    qcsim::DensePlanes p{std::vector<double>(re, re + n), std::vector<double>(im, im + n)};
    return qcsim::planes_sq_norm(p);
}

// Gate kinds in circuit.hpp:36-49 order.
static qcsim::Gate make_gate(int kind, double theta, const int32_t *qs, int nq) {
    qcsim::Gate g{static_cast<qcsim::GateKind>(kind), theta, std::vector<int>(qs, qs + nq)};
    return g;
}

EXPORT int ref_gate_action(int kind, double theta, const int32_t *qs, int nq, qcsim_action *out) {
    return guarded([&] { *out = flatten(qcsim::gate_action(make_gate(kind, theta, qs, nq))); });
}

// Circuits as lowered action arrays.  Pass out = nullptr to query the count.
static int emit_circuit(const qcsim::Circuit &c, qcsim_action *out, uint64_t cap, uint64_t *count) {
    *count = c.gates.size();
    if (!out) return 0;
    if (cap < c.gates.size()) throw std::invalid_argument("output capacity too small");
    for (size_t k = 0; k < c.gates.size(); ++k) out[k] = flatten(qcsim::gate_action(c.gates[k]));
    return 0;
}

EXPORT int ref_build_qft(int n, int swaps, qcsim_action *out, uint64_t cap, uint64_t *count) {
    return guarded([&] { emit_circuit(qcsim::build_qft(n, swaps != 0), out, cap, count); });
}

EXPORT int ref_build_grover(int n, uint64_t marked, int iters, qcsim_action *out, uint64_t cap,
                            uint64_t *count) {
    return guarded([&] { emit_circuit(qcsim::build_grover(n, marked, iters), out, cap, count); });
}

EXPORT int ref_grover_optimal_iterations(int n) { return qcsim::grover_optimal_iterations(n); }

// ---------------------------------------------------------------- engine
namespace {
double tree_sq(const double *re, const double *im, size_t len) {
    if (len == 1) {
        double a = re[0] * re[0], b = im[0] * im[0];
        return a + b;
    }
    size_t h = len / 2;
    double x = tree_sq(re, im, h), y = tree_sq(re + h, im + h, h);
    return x + y;
}
double tree_sum(const double *v, size_t len) {
    if (len == 1) return v[0];
    size_t h = len / 2;
    double a = tree_sum(v, h), b = tree_sum(v + h, h);
    return a + b;
}
inline void cmul(double ar, double ai, double br, double bi, double &cr, double &ci) {
    double t1 = ar * br, t2 = ai * bi, t3 = ar * bi, t4 = ai * br;
    cr = t1 - t2;
    ci = t3 + t4;
}
} // namespace

struct RefEngine {
    int n, s;
    uint64_t S, L;
    qcsim::CodecConfig cfg;
    int norm_every;
    double tol;
    int workers;
    std::vector<qcsim::CompressedPlanes> slices;
    std::vector<double> sq;
    uint64_t gates = 0;
    double rmin = INFINITY, rsum = 0;
    uint64_t calls = 0;
};

EXPORT int ref_engine_create(const qcsim_engine_config *c, int workers, RefEngine **out) {
    return guarded([&] {
        auto *e = new RefEngine();
        e->n = c->num_qubits;
        e->s = c->slice_bits < 0 ? qcsim::default_slice_bits(c->num_qubits) : c->slice_bits;
        e->S = 1ull << (e->n - e->s);
        e->L = 1ull << e->s;
        e->cfg = to_cfg(&c->codec);
        e->cfg.validate();
        e->norm_every = c->norm_every;
        e->tol = c->norm_drift_tolerance;
        e->workers = workers > 0 ? workers : (int)std::max(1u, std::thread::hardware_concurrency());
        e->slices.resize(e->S);
        e->sq.assign(e->S, 0.0);
        *out = e;
    });
}

EXPORT void ref_engine_destroy(RefEngine *e) { delete e; }

template <class F> static void parallel_for(int workers, uint64_t count, F &&f) {
    std::atomic<uint64_t> next{0};
    std::exception_ptr err;
    std::atomic<bool> failed{false};
    auto body = [&] {
        try {
            for (;;) {
                uint64_t j = next.fetch_add(1);
                if (j >= count || failed.load()) return;
                f(j);
            }
        } catch (...) {
            if (!failed.exchange(true)) err = std::current_exception();
        }
    };
    std::vector<std::thread> pool;
    int w = (int)std::min<uint64_t>(workers, count);
    for (int k = 1; k < w; ++k) pool.emplace_back(body);
    body();
    for (auto &t : pool) t.join();
    if (err) std::rethrow_exception(err);
}

EXPORT int ref_engine_load_basis(RefEngine *e, uint64_t x) {
    return guarded([&] {
        if (x >= (1ull << e->n)) throw std::invalid_argument("basis index out of range");
        std::vector<double> stats(2 * e->S);
        parallel_for(e->workers, e->S, [&](uint64_t j) {
            std::vector<double> re(e->L, 0.0), im(e->L, 0.0);
            if (j == (x >> e->s)) re[x & (e->L - 1)] = 1.0;
            e->sq[j] = tree_sq(re.data(), im.data(), e->L);
            auto [br, sr] = qcsim::compress_plane(re, e->cfg);
            auto [bi, si] = qcsim::compress_plane(im, e->cfg);
            e->slices[j] = qcsim::CompressedPlanes{std::move(br), std::move(bi)};
            stats[2 * j] = sr.ratio;
            stats[2 * j + 1] = si.ratio;
        });
        for (double r : stats) {
            e->rmin = std::min(e->rmin, r);
            e->rsum += r;
            e->calls++;
        }
    });
}

static uint64_t partner_of(const qcsim_action &a, int s, uint64_t j) {
    if (a.kind == QCSIM_ACTION_BUTTERFLY && a.target >= s) return j ^ (1ull << (a.target - s));
    if (a.kind == QCSIM_ACTION_SWAP) {
        uint64_t hm = 0;
        if (a.a >= s) hm |= 1ull << (a.a - s);
        if (a.b >= s) hm |= 1ull << (a.b - s);
        return j ^ hm;
    }
    return j;
}

// One gate pass over slices [first, first+count) (count = S for a full
// pass; the CPU baseline times bounded samples of slices).
EXPORT int ref_engine_gate(RefEngine *e, const qcsim_action *act, uint64_t first, uint64_t count) {
    return guarded([&] {
        const qcsim_action &a = *act;
        bool apply = e->norm_every > 0 && (e->gates % (uint64_t)e->norm_every) == 0;
        double scale = 1.0;
        if (apply) {
            double G = tree_sum(e->sq.data(), e->S);
            if (!std::isfinite(G) || std::fabs(G - 1.0) > 10.0 * e->tol)
                throw qcsim::NumericError("norm drift before gate " + std::to_string(e->gates));
            scale = 1.0 / std::sqrt(G);
        }
        std::vector<qcsim::CompressedPlanes> out(count);
        std::vector<double> nsq(count), stats(2 * count);
        parallel_for(e->workers, count, [&](uint64_t k) {
            uint64_t j = first + k;
            uint64_t pj = partner_of(a, e->s, j);
            qcsim::DensePlanes own = qcsim::slice_planes(qcsim::Slice{j, e->slices[j], 0.0});
            qcsim::DensePlanes par;
            if (pj != j) par = qcsim::slice_planes(qcsim::Slice{pj, e->slices[pj], 0.0});
            if (apply) {
                for (uint64_t i = 0; i < e->L; ++i) {
                    own.re[i] = own.re[i] * scale;
                    own.im[i] = own.im[i] * scale;
                }
                if (pj != j)
                    for (uint64_t i = 0; i < e->L; ++i) {
                        par.re[i] = par.re[i] * scale;
                        par.im[i] = par.im[i] * scale;
                    }
            }
            auto fetch = [&](uint64_t g, double &r, double &im) {
                const qcsim::DensePlanes &src = (g >> e->s) == j ? own : par;
                uint64_t off = g & (e->L - 1);
                r = src.re[off];
                im = src.im[off];
            };
            std::vector<double> nre(e->L), nim(e->L);
            for (uint64_t i = 0; i < e->L; ++i) {
                uint64_t g = (j << e->s) | i;
                double vr, vi;
                if (a.kind == QCSIM_ACTION_DIAGONAL) {
                    fetch(g, vr, vi);
                    if ((g & a.mask) == a.mask) cmul(a.factor[0], a.factor[1], vr, vi, nre[i], nim[i]);
                    else { nre[i] = vr; nim[i] = vi; }
                } else if (a.kind == QCSIM_ACTION_BUTTERFLY) {
                    if ((g & a.mask) != a.mask) { fetch(g, nre[i], nim[i]); continue; }
                    uint64_t tb = 1ull << a.target;
                    double v0r, v0i, v1r, v1i, p0r, p0i, p1r, p1i;
                    fetch(g & ~tb, v0r, v0i);
                    fetch(g | tb, v1r, v1i);
                    const double *u = (g & tb) ? a.u + 4 : a.u;
                    cmul(u[0], u[1], v0r, v0i, p0r, p0i);
                    cmul(u[2], u[3], v1r, v1i, p1r, p1i);
                    nre[i] = p0r + p1r;
                    nim[i] = p0i + p1i;
                } else {
                    uint64_t ba = (g >> a.a) & 1, bb = (g >> a.b) & 1;
                    uint64_t src = ba != bb ? g ^ ((1ull << a.a) | (1ull << a.b)) : g;
                    fetch(src, nre[i], nim[i]);
                }
            }
            nsq[k] = tree_sq(nre.data(), nim.data(), e->L);
            auto [br, sr] = qcsim::compress_plane(nre, e->cfg);
            auto [bi, si] = qcsim::compress_plane(nim, e->cfg);
            out[k] = qcsim::CompressedPlanes{std::move(br), std::move(bi)};
            stats[2 * k] = sr.ratio;
            stats[2 * k + 1] = si.ratio;
        });
        for (uint64_t k = 0; k < count; ++k) {
            e->slices[first + k] = std::move(out[k]);
            e->sq[first + k] = nsq[k];
        }
        for (double r : stats) {
            e->rmin = std::min(e->rmin, r);
            e->rsum += r;
            e->calls++;
        }
        e->gates++;
    });
}

EXPORT int ref_engine_export_blocks(RefEngine *e, uint8_t *out, uint64_t cap, uint64_t *len) {
    return guarded([&] {
        std::vector<uint8_t> all;
        for (auto &sl : e->slices) {
            sl.re.append_bytes(all);
            sl.im.append_bytes(all);
        }
        *len = all.size();
        if (out) {
            if (all.size() > cap) throw std::invalid_argument("output capacity too small");
            std::memcpy(out, all.data(), all.size());
        }
    });
}

EXPORT int ref_engine_metrics(RefEngine *e, qcsim_run_metrics *m) {
    std::memset(m, 0, sizeof *m);
    m->min_compression_ratio = e->calls ? e->rmin : 0.0;
    m->mean_compression_ratio = e->calls ? e->rsum / (double)e->calls : 0.0;
    m->final_norm = tree_sum(e->sq.data(), e->S);
    m->compress_calls = e->calls;
    m->gates = e->gates;
    m->dense_bytes = 16ull << e->n;
    return 0;
}
