// qcsim_api.cpp -- host C++ implementation of the qcsim API (include/qcsim/)
// on top of the C-ABI (include/qcsim_c.h, libqcsim_b200.so).
//
// Codec and engine calls go to the GPU; the remaining API surface of the
// reference (statevec container, circuit IR / text format, dense reference
// simulator) is host-side, as it is upstream.  Behaviour and messages follow
// the reference lines cited per function.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <istream>
#include <numbers>
#include <ostream>
#include <set>
#include <sstream>
#include <stdexcept>

#include "qcsim/circuit.hpp"
#include "qcsim/codec.hpp"
#include "qcsim/engine.hpp"
#include "qcsim/errors.hpp"
#include "qcsim/reference.hpp"
#include "qcsim/statevec.hpp"
#include "qcsim_c.h"

namespace qcsim {
namespace {

// qcsim_status -> the reference exception taxonomy (errors.hpp:24-51)
void check(qcsim_status st) {
    if (st == QCSIM_OK) return;
    const std::string msg = qcsim_last_error();
    switch (st) {
    case QCSIM_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QCSIM_CODEC: throw CodecError(msg);
    case QCSIM_CAPACITY: throw CapacityError(msg);
    case QCSIM_PARSE: throw ParseError(0, msg);
    case QCSIM_NUMERIC: throw NumericError(msg);
    case QCSIM_NOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
    }
}

qcsim_codec_config to_c(const CodecConfig &c) {
    qcsim_codec_config o{};
    o.mode = static_cast<uint8_t>(c.mode);
    o.predictor = static_cast<uint8_t>(c.predictor);
    o.quant_code_bits = c.quant_code_bits;
    o.bound = c.bound;
    return o;
}

void le_put(std::vector<uint8_t> &out, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
uint64_t le_get(std::span<const uint8_t> b, size_t at, int bytes) {
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[at + static_cast<size_t>(i)];
    return v;
}

qcsim_action to_c(const GateAction &ga) {
    qcsim_action a{};
    if (const auto *d = std::get_if<DiagonalOp>(&ga)) {
        a.kind = QCSIM_ACTION_DIAGONAL;
        a.mask = d->mask;
        a.factor[0] = d->factor.real();
        a.factor[1] = d->factor.imag();
    } else if (const auto *b = std::get_if<ButterflyOp>(&ga)) {
        a.kind = QCSIM_ACTION_BUTTERFLY;
        a.target = b->target;
        a.mask = b->control_mask;
        const Amplitude u[4] = {b->u.u00, b->u.u01, b->u.u10, b->u.u11};
        for (int k = 0; k < 4; ++k) {
            a.u[2 * k] = u[k].real();
            a.u[2 * k + 1] = u[k].imag();
        }
    } else {
        const auto &s = std::get<SwapOp>(ga);
        a.kind = QCSIM_ACTION_SWAP;
        a.a = s.a;
        a.b = s.b;
    }
    return a;
}

// DESIGN.md §3 product order: (a+bi)(c+di) = (ac - bd) + (ad + bc)i
Amplitude cmul(Amplitude f, Amplitude v) {
    const double t1 = f.real() * v.real(), t2 = f.imag() * v.imag();
    const double t3 = f.real() * v.imag(), t4 = f.imag() * v.real();
    return {t1 - t2, t3 + t4};
}

} // namespace

// ------------------------------------------------------------------ codec
void CodecConfig::validate() const { // codec.cpp:331-341
    const qcsim_codec_config c = to_c(*this);
    check(qcsim_codec_validate(&c));
}

void CompressedBlock::append_bytes(std::vector<uint8_t> &out) const { // codec.cpp:343-357
    out.insert(out.end(), {'Q', 'C', 'B', '1', kFormatVersion, static_cast<uint8_t>(mode),
                           static_cast<uint8_t>(predictor), quant_code_bits});
    le_put(out, element_count, 8);
    le_put(out, std::bit_cast<uint64_t>(effective_abs_bound), 8);
    le_put(out, outlier_count, 8);
    le_put(out, payload.size(), 8);
    out.insert(out.end(), payload.begin(), payload.end());
}

std::vector<uint8_t> CompressedBlock::to_bytes() const {
    std::vector<uint8_t> out;
    out.reserve(byte_size());
    append_bytes(out);
    return out;
}

CompressedBlock CompressedBlock::from_bytes(std::span<const uint8_t> b, size_t *consumed) { // codec.cpp:366-408
    if (b.size() < kHeaderBytes) throw CodecError("block header truncated");
    if (!(b[0] == 'Q' && b[1] == 'C' && b[2] == 'B' && b[3] == '1')) throw CodecError("bad block magic");
    if (b[4] != kFormatVersion) throw CodecError("unsupported block version " + std::to_string(b[4]));
    if (b[5] > 2) throw CodecError("bad codec mode byte");
    if (b[6] > 1) throw CodecError("bad predictor byte");
    CompressedBlock blk;
    blk.mode = static_cast<CodecMode>(b[5]);
    blk.predictor = static_cast<Predictor>(b[6]);
    blk.quant_code_bits = b[7];
    if (blk.quant_code_bits < 4 || blk.quant_code_bits > 24) throw CodecError("quant_code_bits out of range");
    blk.element_count = le_get(b, 8, 8);
    blk.effective_abs_bound = std::bit_cast<double>(le_get(b, 16, 8));
    blk.outlier_count = le_get(b, 24, 8);
    const uint64_t plen = le_get(b, 32, 8);
    if (blk.element_count == 0) throw CodecError("element_count must be at least 1");
    if (blk.outlier_count > blk.element_count) throw CodecError("outlier_count exceeds element_count");
    if (!(blk.effective_abs_bound >= 0.0) || !std::isfinite(blk.effective_abs_bound))
        throw CodecError("bad effective_abs_bound");
    if (plen > b.size() - kHeaderBytes) throw CodecError("block payload truncated");
    blk.payload.assign(b.begin() + kHeaderBytes, b.begin() + kHeaderBytes + static_cast<size_t>(plen));
    if (consumed) *consumed = kHeaderBytes + static_cast<size_t>(plen);
    return blk;
}

std::pair<CompressedBlock, CodecStats> compress_plane(std::span<const double> values, const CodecConfig &config) {
    const qcsim_codec_config c = to_c(config);
    std::vector<uint8_t> out(qcsim_block_bound(std::max<size_t>(values.size(), 1), config.quant_code_bits));
    uint64_t len = 0;
    qcsim_codec_stats st{};
    check(qcsim_compress_plane(values.data(), values.size(), &c, out.data(), out.size(), &len, &st));
    CompressedBlock blk = CompressedBlock::from_bytes(std::span<const uint8_t>(out.data(), len));
    return {std::move(blk), CodecStats{st.input_bytes, st.output_bytes, st.ratio, st.outlier_fraction}};
}

std::vector<double> decompress_plane(const CompressedBlock &block) {
    const std::vector<uint8_t> bytes = block.to_bytes();
    uint64_t n = 0;
    check(qcsim_decompress_plane(bytes.data(), bytes.size(), nullptr, 0, &n, nullptr));
    std::vector<double> out(n);
    check(qcsim_decompress_plane(bytes.data(), bytes.size(), out.data(), out.size(), &n, nullptr));
    return out;
}

// --------------------------------------------------------------- statevec
namespace {
struct Kahan { // statevec.cpp:32-45
    double sum = 0.0, carry = 0.0;
    void add(double x) {
        const double y = x - carry;
        const double t = sum + y;
        carry = (t - sum) - y;
        sum = t;
    }
};
void check_qubits(int n) {
    if (n < 1 || n > 62) throw std::invalid_argument("qubit count must be in [1, 62]");
}
void check_slice_bits(int n, int s) {
    if (s < 0 || s > n) throw std::invalid_argument("slice_bits must be in [0, num_qubits]");
}
} // namespace

DensePlanes slice_planes(const Slice &slice) {
    if (slice.is_dense()) return slice.dense();
    return DensePlanes{decompress_plane(slice.blocks().re), decompress_plane(slice.blocks().im)};
}

double planes_sq_norm(const DensePlanes &p) {
    Kahan k;
    for (size_t i = 0; i < p.size(); ++i) k.add(p.re[i] * p.re[i] + p.im[i] * p.im[i]);
    return k.sum;
}

StateVector::StateVector(int num_qubits, int slice_bits) : num_qubits_(num_qubits), slice_bits_(slice_bits) {
    check_qubits(num_qubits);
    check_slice_bits(num_qubits, slice_bits);
    const uint64_t count = uint64_t{1} << (num_qubits - slice_bits);
    slices_.resize(count);
    for (uint64_t j = 0; j < count; ++j) {
        slices_[j].index = j;
        slices_[j].payload = DensePlanes{std::vector<double>(slice_size()), std::vector<double>(slice_size())};
    }
}

Amplitude StateVector::amplitude(uint64_t g) const {
    if (g >= num_amplitudes()) throw std::invalid_argument("amplitude index out of range");
    const Slice &sl = slices_[slice_of_index(g, slice_bits_)];
    const uint64_t k = offset_of_index(g, slice_bits_);
    if (sl.is_dense()) return {sl.dense().re[k], sl.dense().im[k]};
    const DensePlanes p = slice_planes(sl);
    return {p.re[k], p.im[k]};
}

StateVector init_basis_state(int n, uint64_t x, int s) {
    check_qubits(n);
    if (s < 0) s = default_slice_bits(n);
    check_slice_bits(n, s);
    if (x >= (uint64_t{1} << n)) throw std::invalid_argument("basis index out of range");
    StateVector st(n, s);
    Slice &sl = st.slices()[slice_of_index(x, s)];
    sl.dense().re[offset_of_index(x, s)] = 1.0;
    sl.sq_norm = 1.0;
    return st;
}

StateVector state_from_amplitudes(int n, std::span<const Amplitude> amps, int s) {
    check_qubits(n);
    if (s < 0) s = default_slice_bits(n);
    check_slice_bits(n, s);
    if (amps.size() != (uint64_t{1} << n)) throw std::invalid_argument("amplitude count must be 2^n");
    StateVector st(n, s);
    for (Slice &sl : st.slices()) {
        const uint64_t base = sl.index << s;
        for (uint64_t k = 0; k < st.slice_size(); ++k) {
            sl.dense().re[k] = amps[base + k].real();
            sl.dense().im[k] = amps[base + k].imag();
        }
        sl.sq_norm = planes_sq_norm(sl.dense());
    }
    return st;
}

std::vector<Amplitude> to_amplitudes(const StateVector &st, int guard) {
    if (st.num_qubits() > guard)
        throw CapacityError("dense materialization of " + std::to_string(st.num_qubits()) + " qubits exceeds the " +
                            std::to_string(guard) + "-qubit guard");
    std::vector<Amplitude> out(st.num_amplitudes());
    for (const Slice &sl : st.slices()) {
        const DensePlanes p = slice_planes(sl);
        const uint64_t base = sl.index << st.slice_bits();
        for (uint64_t k = 0; k < st.slice_size(); ++k) out[base + k] = {p.re[k], p.im[k]};
    }
    return out;
}

double global_sq_norm(const StateVector &st) {
    Kahan k;
    for (const Slice &sl : st.slices()) {
        const DensePlanes p = slice_planes(sl);
        for (size_t i = 0; i < p.size(); ++i) k.add(p.re[i] * p.re[i] + p.im[i] * p.im[i]);
    }
    return k.sum;
}

Amplitude inner_product(const StateVector &a, const StateVector &b) { // statevec.cpp:199-242: conj(a).b
    if (a.num_qubits() != b.num_qubits()) throw std::invalid_argument("inner product dimension mismatch");
    const bool a_fine = a.slice_bits() <= b.slice_bits();
    const StateVector &fine = a_fine ? a : b;
    const StateVector &coarse = a_fine ? b : a;
    const uint64_t fsz = fine.slice_size(), per = coarse.slice_size() / fsz;
    Kahan re, im;
    for (const Slice &cs : coarse.slices()) {
        const DensePlanes cp = slice_planes(cs);
        for (uint64_t f = 0; f < per; ++f) {
            const DensePlanes fp = slice_planes(fine.slices()[cs.index * per + f]);
            for (uint64_t k = 0; k < fsz; ++k) {
                const double xr = a_fine ? fp.re[k] : cp.re[f * fsz + k];
                const double xi = a_fine ? fp.im[k] : cp.im[f * fsz + k];
                const double yr = a_fine ? cp.re[f * fsz + k] : fp.re[k];
                const double yi = a_fine ? cp.im[f * fsz + k] : fp.im[k];
                re.add(xr * yr + xi * yi);
                im.add(xr * yi - xi * yr);
            }
        }
    }
    return {re.sum, im.sum};
}

double fidelity(const StateVector &a, const StateVector &b) {
    const Amplitude ip = inner_product(a, b);
    return ip.real() * ip.real() + ip.imag() * ip.imag();
}

void write_state_dump(const StateVector &st, std::ostream &out) { // statevec.cpp:249-263, "QSV1"
    std::vector<uint8_t> hdr = {'Q', 'S', 'V', '1'};
    le_put(hdr, static_cast<uint32_t>(st.num_qubits()), 4);
    le_put(hdr, 0, 8);
    out.write(reinterpret_cast<const char *>(hdr.data()), hdr.size());
    std::vector<uint8_t> buf;
    for (const Slice &sl : st.slices()) {
        const DensePlanes p = slice_planes(sl);
        buf.clear();
        for (size_t k = 0; k < p.size(); ++k) {
            le_put(buf, std::bit_cast<uint64_t>(p.re[k]), 8);
            le_put(buf, std::bit_cast<uint64_t>(p.im[k]), 8);
        }
        out.write(reinterpret_cast<const char *>(buf.data()), buf.size());
    }
    if (!out) throw std::runtime_error("state dump write failed");
}

StateVector read_state_dump(std::istream &in, int s) { // statevec.cpp:265-293
    uint8_t hdr[16];
    in.read(reinterpret_cast<char *>(hdr), 4);
    if (!in || std::memcmp(hdr, "QSV1", 4) != 0) throw std::runtime_error("not a state dump (bad magic)");
    in.read(reinterpret_cast<char *>(hdr + 4), 12);
    const uint64_t n = le_get(std::span<const uint8_t>(hdr, 16), 4, 4);
    if (!in || n < 1 || n > 62) throw std::runtime_error("state dump header corrupt");
    const int nq = static_cast<int>(n);
    if (s < 0) s = default_slice_bits(nq);
    check_slice_bits(nq, s);
    StateVector st(nq, s);
    std::vector<uint8_t> buf(16 * st.slice_size());
    for (Slice &sl : st.slices()) {
        in.read(reinterpret_cast<char *>(buf.data()), static_cast<std::streamsize>(buf.size()));
        if (!in) throw std::runtime_error("state dump truncated");
        const std::span<const uint8_t> b(buf);
        for (uint64_t k = 0; k < st.slice_size(); ++k) {
            sl.dense().re[k] = std::bit_cast<double>(le_get(b, 16 * k, 8));
            sl.dense().im[k] = std::bit_cast<double>(le_get(b, 16 * k + 8, 8));
        }
        sl.sq_norm = planes_sq_norm(sl.dense());
    }
    return st;
}

// ---------------------------------------------------------------- circuit
namespace {
size_t arity(GateKind k) {
    switch (k) {
    case GateKind::CPhase:
    case GateKind::CNOT:
    case GateKind::CZ:
    case GateKind::Swap: return 2;
    case GateKind::MCZ: return 0;
    default: return 1;
    }
}
void validate_gate(const Gate &g, int n) { // circuit.cpp:51-69
    if (g.kind == GateKind::MCZ) {
        if (g.qubits.empty()) throw std::invalid_argument("mcz needs at least one qubit");
    } else if (g.qubits.size() != arity(g.kind)) {
        throw std::invalid_argument("wrong qubit count for gate");
    }
    std::set<int> seen;
    for (int q : g.qubits) {
        if (q < 0 || q >= n) throw std::invalid_argument("qubit index " + std::to_string(q) + " out of range");
        if (!seen.insert(q).second) throw std::invalid_argument("duplicate qubit index in gate");
    }
    if (!std::isfinite(g.theta)) throw std::invalid_argument("gate angle must be finite");
}
constexpr double kInvSqrt2 = 0.7071067811865475244;
} // namespace

void validate_circuit(const Circuit &c) {
    if (c.num_qubits < 1) throw std::invalid_argument("circuit needs at least one qubit");
    for (const Gate &g : c.gates) validate_gate(g, c.num_qubits);
}

Circuit build_qft(int n, bool swaps) { // circuit.cpp:88-104
    if (n < 1) throw std::invalid_argument("QFT needs at least one qubit");
    Circuit c{n, "qft" + std::to_string(n), {}};
    for (int i = n - 1; i >= 0; --i) {
        c.gates.push_back(Gate::h(i));
        for (int j = i - 1; j >= 0; --j) c.gates.push_back(Gate::cphase(std::numbers::pi / std::ldexp(1.0, i - j), j, i));
    }
    if (swaps)
        for (int i = 0; i < n / 2; ++i) c.gates.push_back(Gate::swap(i, n - 1 - i));
    return c;
}

Circuit build_grover_oracle(int n, uint64_t marked) { // circuit.cpp:106-125
    if (n < 2) throw std::invalid_argument("Grover search needs at least two qubits");
    if (marked >= (uint64_t{1} << n)) throw std::invalid_argument("marked state out of range");
    Circuit c{n, "grover_oracle", {}};
    std::vector<int> all;
    for (int q = 0; q < n; ++q) all.push_back(q);
    for (int pass = 0; pass < 2; ++pass) {
        for (int q = 0; q < n; ++q)
            if (!((marked >> q) & 1)) c.gates.push_back(Gate::x(q));
        if (pass == 0) c.gates.push_back(Gate::mcz(all));
    }
    return c;
}

Circuit build_grover(int n, uint64_t marked, int iterations) { // circuit.cpp:127-160
    if (n < 2) throw std::invalid_argument("Grover search needs at least two qubits");
    if (marked >= (uint64_t{1} << n)) throw std::invalid_argument("marked state out of range");
    if (iterations < 1) throw std::invalid_argument("iterations must be at least 1");
    Circuit c{n, "grover" + std::to_string(n), {}};
    std::vector<int> all;
    for (int q = 0; q < n; ++q) all.push_back(q);
    auto layer = [&](Gate (*make)(int)) {
        for (int q = 0; q < n; ++q) c.gates.push_back(make(q));
    };
    layer(&Gate::h);
    const Circuit oracle = build_grover_oracle(n, marked);
    for (int it = 0; it < iterations; ++it) {
        c.gates.insert(c.gates.end(), oracle.gates.begin(), oracle.gates.end());
        layer(&Gate::h);
        layer(&Gate::x);
        c.gates.push_back(Gate::mcz(all));
        layer(&Gate::x);
        layer(&Gate::h);
    }
    return c;
}

int grover_optimal_iterations(int n) { // circuit.cpp:162-168
    if (n < 2) throw std::invalid_argument("Grover search needs at least two qubits");
    const double r = std::floor(std::numbers::pi / 4.0 * std::sqrt(std::ldexp(1.0, n)));
    return r < 1.0 ? 1 : static_cast<int>(r);
}

Circuit parse_circuit(const std::string &text) { // circuit.cpp:222-314, format SPEC.md:288
    Circuit c;
    bool header = false;
    std::istringstream in(text);
    std::string raw;
    int line = 0;
    while (std::getline(in, raw)) {
        ++line;
        if (const auto h = raw.find('#'); h != std::string::npos) raw.erase(h);
        std::vector<std::string> f;
        std::istringstream fs(raw);
        for (std::string w; fs >> w;) f.push_back(w);
        if (f.empty()) continue;
        auto fail = [&](const std::string &m) -> void { throw ParseError(line, m); };
        auto need = [&](size_t k) {
            if (f.size() - 1 != k)
                fail("gate '" + f[0] + "' expects " + std::to_string(k) + " argument(s), got " +
                     std::to_string(f.size() - 1));
        };
        auto qubit = [&](size_t i) {
            size_t used = 0;
            long v = 0;
            try {
                v = std::stol(f[i], &used);
            } catch (const std::exception &) {
                fail("malformed qubit index '" + f[i] + "'");
            }
            if (used != f[i].size() || v < 0) fail("malformed qubit index '" + f[i] + "'");
            if (v >= c.num_qubits)
                fail("qubit index " + f[i] + " out of range for width " + std::to_string(c.num_qubits));
            return static_cast<int>(v);
        };
        auto angle = [&](size_t i) {
            size_t used = 0;
            double v = 0.0;
            try {
                v = std::stod(f[i], &used);
            } catch (const std::exception &) {
                fail("malformed angle '" + f[i] + "'");
            }
            if (used != f[i].size() || !std::isfinite(v)) fail("malformed angle '" + f[i] + "'");
            return v;
        };
        const std::string &op = f[0];
        if (!header) {
            if (op != "qubits") fail("expected 'qubits <n>' header before gates");
            need(1);
            size_t used = 0;
            long n = 0;
            try {
                n = std::stol(f[1], &used);
            } catch (const std::exception &) {
                fail("malformed qubit count '" + f[1] + "'");
            }
            if (used != f[1].size() || n < 1 || n > 62) fail("qubit count must be in [1, 62]");
            c.num_qubits = static_cast<int>(n);
            header = true;
            continue;
        }
        if (op == "qubits") fail("duplicate 'qubits' header");
        Gate g{GateKind::H, 0.0, {}};
        static const std::pair<const char *, GateKind> one[] = {{"h", GateKind::H}, {"x", GateKind::X},
                                                                {"y", GateKind::Y}, {"z", GateKind::Z},
                                                                {"s", GateKind::S}, {"t", GateKind::T}};
        bool done = false;
        for (const auto &[name, kind] : one)
            if (op == name) {
                need(1);
                g = Gate{kind, 0.0, {qubit(1)}};
                done = true;
            }
        if (done) {
        } else if (op == "p") {
            need(2);
            g = Gate::phase(angle(1), qubit(2));
        } else if (op == "cp") {
            need(3);
            g = Gate::cphase(angle(1), qubit(2), qubit(3));
        } else if (op == "cx") {
            need(2);
            g = Gate::cnot(qubit(1), qubit(2));
        } else if (op == "cz") {
            need(2);
            g = Gate::cz(qubit(1), qubit(2));
        } else if (op == "swap") {
            need(2);
            g = Gate::swap(qubit(1), qubit(2));
        } else if (op == "mcz") {
            if (f.size() < 2) fail("mcz needs at least one qubit");
            std::vector<int> qs;
            for (size_t i = 1; i < f.size(); ++i) qs.push_back(qubit(i));
            g = Gate::mcz(std::move(qs));
        } else {
            fail("unknown gate '" + op + "'");
        }
        try {
            validate_gate(g, c.num_qubits);
        } catch (const std::invalid_argument &e) {
            fail(e.what());
        }
        c.gates.push_back(std::move(g));
    }
    if (!header) throw ParseError(line == 0 ? 1 : line, "missing 'qubits <n>' header");
    return c;
}

std::string render_circuit(const Circuit &c) { // circuit.cpp:316-364
    std::ostringstream out;
    out << "qubits " << c.num_qubits << "\n";
    auto ang = [](double t) {
        char b[32];
        std::snprintf(b, sizeof b, "%.17g", t);
        return std::string(b);
    };
    static const char *names[] = {"h", "x", "y", "z", "s", "t"};
    for (const Gate &g : c.gates) {
        switch (g.kind) {
        case GateKind::Phase: out << "p " << ang(g.theta) << " " << g.target(); break;
        case GateKind::CPhase: out << "cp " << ang(g.theta) << " " << g.control() << " " << g.target(); break;
        case GateKind::CNOT: out << "cx " << g.control() << " " << g.target(); break;
        case GateKind::CZ: out << "cz " << g.control() << " " << g.target(); break;
        case GateKind::Swap: out << "swap " << g.qubits[0] << " " << g.qubits[1]; break;
        case GateKind::MCZ:
            out << "mcz";
            for (int q : g.qubits) out << " " << q;
            break;
        default: out << names[static_cast<int>(g.kind)] << " " << g.target();
        }
        out << "\n";
    }
    return out.str();
}

Mat2 unitary2(GateKind k, double theta) { // circuit.cpp:366-390
    const double r = kInvSqrt2;
    switch (k) {
    case GateKind::H: return {{r, 0}, {r, 0}, {r, 0}, {-r, 0}};
    case GateKind::X: return {{0, 0}, {1, 0}, {1, 0}, {0, 0}};
    case GateKind::Y: return {{0, 0}, {0, -1}, {0, 1}, {0, 0}};
    case GateKind::Z: return {{1, 0}, {0, 0}, {0, 0}, {-1, 0}};
    case GateKind::S: return {{1, 0}, {0, 0}, {0, 0}, {0, 1}};
    case GateKind::T: return {{1, 0}, {0, 0}, {0, 0}, {r, r}};
    case GateKind::Phase: return {{1, 0}, {0, 0}, {0, 0}, {std::cos(theta), std::sin(theta)}};
    default: throw std::invalid_argument("gate kind has no single-qubit matrix");
    }
}

GateAction gate_action(const Gate &g) { // circuit.cpp:392-427
    const auto bit = [](int q) { return uint64_t{1} << q; };
    switch (g.kind) {
    case GateKind::H:
    case GateKind::X:
    case GateKind::Y: return ButterflyOp{unitary2(g.kind), g.target(), 0};
    case GateKind::Z: return DiagonalOp{bit(g.target()), {-1.0, 0.0}};
    case GateKind::S: return DiagonalOp{bit(g.target()), {0.0, 1.0}};
    case GateKind::T: return DiagonalOp{bit(g.target()), {kInvSqrt2, kInvSqrt2}};
    case GateKind::Phase: return DiagonalOp{bit(g.target()), {std::cos(g.theta), std::sin(g.theta)}};
    case GateKind::CPhase:
        return DiagonalOp{bit(g.control()) | bit(g.target()), {std::cos(g.theta), std::sin(g.theta)}};
    case GateKind::CNOT: return ButterflyOp{unitary2(GateKind::X), g.target(), bit(g.control())};
    case GateKind::CZ: return DiagonalOp{bit(g.control()) | bit(g.target()), {-1.0, 0.0}};
    case GateKind::Swap: return SwapOp{g.qubits[0], g.qubits[1]};
    case GateKind::MCZ: {
        uint64_t m = 0;
        for (int q : g.qubits) m |= bit(q);
        return DiagonalOp{m, {-1.0, 0.0}};
    }
    }
    throw std::invalid_argument("unknown gate kind");
}

// -------------------------------------------------------------- reference
DenseState make_dense_basis(int n, uint64_t x) {
    check_qubits(n);
    if (x >= (uint64_t{1} << n)) throw std::invalid_argument("basis index out of range");
    DenseState d{n, std::vector<Amplitude>(uint64_t{1} << n)};
    d.amps[x] = 1.0;
    return d;
}

void apply_action_dense(const GateAction &ga, std::vector<Amplitude> &amps) {
    const uint64_t N = amps.size();
    if (const auto *d = std::get_if<DiagonalOp>(&ga)) {
        for (uint64_t g = 0; g < N; ++g)
            if ((g & d->mask) == d->mask) amps[g] = cmul(d->factor, amps[g]);
    } else if (const auto *b = std::get_if<ButterflyOp>(&ga)) {
        const uint64_t tb = uint64_t{1} << b->target;
        for (uint64_t g0 = 0; g0 < N; ++g0) {
            if ((g0 & tb) || (g0 & b->control_mask) != b->control_mask) continue;
            const Amplitude v0 = amps[g0], v1 = amps[g0 | tb];
            const Amplitude p0 = cmul(b->u.u00, v0), p1 = cmul(b->u.u01, v1);
            const Amplitude p2 = cmul(b->u.u10, v0), p3 = cmul(b->u.u11, v1);
            amps[g0] = {p0.real() + p1.real(), p0.imag() + p1.imag()};
            amps[g0 | tb] = {p2.real() + p3.real(), p2.imag() + p3.imag()};
        }
    } else {
        const auto &s = std::get<SwapOp>(ga);
        const uint64_t ma = uint64_t{1} << s.a, mb = uint64_t{1} << s.b;
        for (uint64_t g = 0; g < N; ++g)
            if ((g & ma) && !(g & mb)) std::swap(amps[g], amps[g ^ ma ^ mb]);
    }
}

DenseState ref_run(const Circuit &c, DenseState st, int guard) {
    if (c.num_qubits > guard)
        throw CapacityError("dense reference run of " + std::to_string(c.num_qubits) + " qubits exceeds the " +
                            std::to_string(guard) + "-qubit guard");
    for (const Gate &g : c.gates) apply_action_dense(gate_action(g), st.amps);
    return st;
}

double success_probability(const DenseState &st, uint64_t x) {
    if (x >= st.amps.size()) throw std::invalid_argument("basis index out of range");
    return st.amps[x].real() * st.amps[x].real() + st.amps[x].imag() * st.amps[x].imag();
}

// ------------------------------------------------------------------ engine
Engine::Engine(int n, const EngineConfig &cfg) : n_(n) {
    qcsim_engine_config c{};
    c.num_qubits = n;
    c.slice_bits = cfg.slice_bits;
    c.codec = to_c(cfg.codec);
    c.compression_enabled = cfg.compression_enabled ? 1 : 0;
    c.norm_every = cfg.norm_policy == NormPolicy::Off ? 0
                   : cfg.norm_policy == NormPolicy::EveryGate ? 1
                                                              : std::max(1, cfg.norm_every_k);
    c.norm_drift_tolerance = cfg.norm_drift_tolerance;
    c.device = cfg.device;
    c.rank = cfg.rank;
    c.world = cfg.world;
    c.wave_bytes = cfg.wave_bytes;
    check(qcsim_engine_create(&c, &h_));
    s_ = cfg.slice_bits < 0 ? default_slice_bits(n) : cfg.slice_bits;
}

Engine::~Engine() {
    if (h_) qcsim_engine_destroy(h_);
}

void Engine::load_basis(uint64_t x) { check(qcsim_engine_load_basis(h_, x)); }

void Engine::load(const StateVector &st) {
    if (st.num_qubits() != n_) throw std::invalid_argument("state width does not match the engine");
    const std::vector<Amplitude> amps = to_amplitudes(st, 62);
    check(qcsim_engine_load_amplitudes(h_, reinterpret_cast<const double *>(amps.data()), amps.size()));
}

RunMetrics Engine::run(const std::vector<GateAction> &actions) {
    std::vector<qcsim_action> acts;
    acts.reserve(actions.size());
    for (const GateAction &a : actions) acts.push_back(to_c(a));
    check(qcsim_engine_run(h_, acts.data(), acts.size(), nullptr));
    return metrics();
}

RunMetrics Engine::run(const Circuit &c) {
    if (c.num_qubits != n_) throw std::invalid_argument("circuit width does not match the engine");
    validate_circuit(c);
    std::vector<GateAction> acts;
    for (const Gate &g : c.gates) acts.push_back(gate_action(g));
    return run(acts);
}

RunMetrics Engine::metrics() const {
    qcsim_run_metrics m{};
    check(qcsim_engine_run(h_, nullptr, 0, &m));
    RunMetrics r;
    r.min_compression_ratio = m.min_compression_ratio;
    r.mean_compression_ratio = m.mean_compression_ratio;
    r.wall_seconds = m.wall_seconds;
    r.peak_compressed_bytes = m.peak_compressed_bytes;
    r.dense_bytes = m.dense_bytes;
    r.final_norm = m.final_norm;
    r.compress_calls = m.compress_calls;
    r.gates = m.gates;
    r.index_bytes = m.index_bytes;
    r.fallback_planes = m.fallback_planes;
    const std::vector<GateMetrics> rows = gate_metrics();
    for (size_t k = 1; k < rows.size(); ++k) r.per_gate_min_ratio.push_back(rows[k].min_ratio);
    return r;
}

std::vector<GateMetrics> Engine::gate_metrics() const {
    uint64_t cnt = 0;
    check(qcsim_engine_gate_metrics(h_, nullptr, 0, &cnt));
    std::vector<qcsim_gate_metrics> raw(cnt);
    check(qcsim_engine_gate_metrics(h_, raw.data(), raw.size(), &cnt));
    std::vector<GateMetrics> out(cnt);
    for (uint64_t k = 0; k < cnt; ++k) {
        out[k].gate_index = (long long)k - 1;
        out[k].min_ratio = raw[k].min_ratio;
        out[k].mean_ratio = raw[k].mean_ratio;
        out[k].seconds = raw[k].seconds;
        out[k].compressed_bytes = raw[k].compressed_bytes;
        out[k].index_bytes = raw[k].index_bytes;
    }
    return out;
}

StateVector Engine::gather_state(int guard) const {
    std::vector<double> buf(uint64_t{2} << n_);
    check(qcsim_engine_gather(h_, buf.data(), buf.size(), guard));
    std::vector<Amplitude> amps(uint64_t{1} << n_);
    for (uint64_t k = 0; k < amps.size(); ++k) amps[k] = {buf[2 * k], buf[2 * k + 1]};
    return state_from_amplitudes(n_, amps, s_);
}

std::vector<CompressedPlanes> Engine::compressed_slices() const {
    uint64_t len = 0;
    const uint64_t P = uint64_t{2} << (n_ - s_);
    std::vector<uint64_t> offs(P + 1);
    check(qcsim_engine_export_blocks(h_, nullptr, 0, &len, offs.data(), offs.size()));
    std::vector<uint8_t> bytes(len);
    check(qcsim_engine_export_blocks(h_, bytes.data(), bytes.size(), &len, offs.data(), offs.size()));
    std::vector<CompressedPlanes> out(P / 2);
    for (uint64_t j = 0; j < P / 2; ++j) {
        out[j].re = CompressedBlock::from_bytes(std::span<const uint8_t>(bytes.data() + offs[2 * j], offs[2 * j + 1] - offs[2 * j]));
        out[j].im = CompressedBlock::from_bytes(
            std::span<const uint8_t>(bytes.data() + offs[2 * j + 1], offs[2 * j + 2] - offs[2 * j + 1]));
    }
    return out;
}

std::vector<double> Engine::slice_norms() const {
    std::vector<double> v(uint64_t{1} << (n_ - s_));
    check(qcsim_engine_slice_norms(h_, v.data(), v.size()));
    return v;
}

void Engine::resume(const std::vector<CompressedPlanes> &slices, const std::vector<double> &sq_norms,
                    uint64_t gates_done) {
    std::vector<uint8_t> bytes;
    std::vector<uint64_t> offs;
    for (const CompressedPlanes &cp : slices) {
        offs.push_back(bytes.size());
        cp.re.append_bytes(bytes);
        offs.push_back(bytes.size());
        cp.im.append_bytes(bytes);
    }
    offs.push_back(bytes.size());
    check(qcsim_engine_load_blocks(h_, bytes.data(), bytes.size(), offs.data(), offs.size() - 1, sq_norms.data(),
                                   sq_norms.size(), gates_done));
}

std::pair<std::unique_ptr<Engine>, RunMetrics> run(const Circuit &c, const EngineConfig &cfg,
                                                   const StateVector &initial) {
    if (initial.num_qubits() != c.num_qubits) throw std::invalid_argument("circuit/state width mismatch");
    EngineConfig e = cfg;
    if (e.slice_bits < 0) e.slice_bits = initial.slice_bits();
    auto eng = std::make_unique<Engine>(c.num_qubits, e);
    eng->load(initial);
    RunMetrics m = eng->run(c);
    return {std::move(eng), m};
}

RunMetrics measure_overhead(const Circuit &c, const EngineConfig &cfg, const StateVector &initial) {
    auto [on, m] = run(c, cfg, initial);
    EngineConfig off_cfg = cfg;
    off_cfg.compression_enabled = false;
    auto [off, moff] = run(c, off_cfg, initial);
    m.baseline_wall_seconds = moff.wall_seconds;
    m.overhead_factor = moff.wall_seconds > 0.0 ? m.wall_seconds / moff.wall_seconds : 0.0;
    return m;
}

namespace {
std::string num(double v) {
    if (!std::isfinite(v)) return "null";
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
} // namespace

std::string metrics_json(const RunMetrics &m, const std::vector<GateMetrics> &rows) {
    std::string o = "{";
    o += "\"min_compression_ratio\": " + num(m.min_compression_ratio);
    o += ", \"mean_compression_ratio\": " + num(m.mean_compression_ratio);
    o += ", \"per_gate_min_ratio\": [";
    for (size_t k = 0; k < m.per_gate_min_ratio.size(); ++k) o += (k ? ", " : "") + num(m.per_gate_min_ratio[k]);
    o += "], \"wall_seconds\": " + num(m.wall_seconds);
    o += ", \"baseline_wall_seconds\": " + (m.baseline_wall_seconds > 0 ? num(m.baseline_wall_seconds) : "null");
    o += ", \"overhead_factor\": " + (m.overhead_factor > 0 ? num(m.overhead_factor) : "null");
    o += ", \"peak_compressed_bytes\": " + std::to_string(m.peak_compressed_bytes);
    o += ", \"dense_bytes\": " + std::to_string(m.dense_bytes);
    o += ", \"final_norm\": " + num(m.final_norm);
    o += ", \"compress_calls\": " + std::to_string(m.compress_calls);
    o += ", \"gates\": " + std::to_string(m.gates);
    o += ", \"index_bytes\": " + std::to_string(m.index_bytes);
    o += ", \"fallback_planes\": " + std::to_string(m.fallback_planes);
    o += ", \"per_gate\": [";
    for (size_t k = 0; k < rows.size(); ++k) {
        const GateMetrics &r = rows[k];
        o += std::string(k ? ", " : "") + "{\"gate_index\": " + std::to_string(r.gate_index) +
             ", \"min_ratio\": " + num(r.min_ratio) + ", \"mean_ratio\": " + num(r.mean_ratio) +
             ", \"seconds\": " + num(r.seconds) + ", \"compressed_bytes\": " + std::to_string(r.compressed_bytes) +
             ", \"index_bytes\": " + std::to_string(r.index_bytes) + "}";
    }
    o += "]}";
    return o;
}

std::string metrics_csv(const std::vector<GateMetrics> &rows) {
    std::string o = "gate_index,min_ratio,mean_ratio,seconds\n";
    for (const GateMetrics &r : rows)
        o += std::to_string(r.gate_index) + "," + num(r.min_ratio) + "," + num(r.mean_ratio) + "," + num(r.seconds) + "\n";
    return o;
}

} // namespace qcsim
