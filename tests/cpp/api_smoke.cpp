// api_smoke.cpp -- the reference's C++ API (include/qcsim/) linked against
// libqcsim.so -> libqcsim_b200.so.  Exercises the drop-in surface the way a
// reference user would: codec round trip, block wire format, builders,
// lowering, the dense reference and the GPU engine (QFT closed form).
// Prints "api_smoke ok" and exits 0 on success.
#include <cmath>
#include <complex>
#include <cstdio>
#include <numbers>
#include <sstream>
#include <vector>

#include "qcsim/circuit.hpp"
#include "qcsim/codec.hpp"
#include "qcsim/engine.hpp"
#include "qcsim/errors.hpp"
#include "qcsim/reference.hpp"
#include "qcsim/statevec.hpp"

#define REQUIRE(c)                                                                                                     \
    do {                                                                                                               \
        if (!(c)) {                                                                                                    \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);                                        \
            return 1;                                                                                                  \
        }                                                                                                              \
    } while (0)

int main() {
    using namespace qcsim;
    // codec (SURVEY.md Appendix A.4 known answer)
    std::vector<double> v{0, 0, 0, 0, 0, 0, 6e-5, 1.0};
    CodecConfig cfg{CodecMode::Absolute, 1e-5, 16, Predictor::PreviousValue};
    auto [blk, st] = compress_plane(v, cfg);
    REQUIRE(blk.byte_size() == 82);
    REQUIRE(std::fabs(compression_ratio(st) - 64.0 / 82.0) < 1e-15);
    const auto bytes = blk.to_bytes();
    size_t used = 0;
    CompressedBlock back = CompressedBlock::from_bytes(bytes, &used);
    REQUIRE(used == 82 && back.payload == blk.payload);
    const auto dec = decompress_plane(back);
    REQUIRE(dec.size() == 8 && dec[6] == 6.000000000000001e-05 && dec[7] == 1.0);
    bool threw = false;
    try {
        CompressedBlock::from_bytes(std::vector<uint8_t>(10));
    } catch (const CodecError &) {
        threw = true;
    }
    REQUIRE(threw);
    threw = false;
    try {
        compress_plane(std::vector<double>{}, cfg);
    } catch (const std::invalid_argument &) {
        threw = true;
    }
    REQUIRE(threw);
    // builders / lowering / text format
    REQUIRE(grover_optimal_iterations(2) == 1 && grover_optimal_iterations(4) == 3 &&
            grover_optimal_iterations(10) == 25);
    const Circuit qft = build_qft(10);
    REQUIRE(qft.gate_count() == 10 + 45 + 5);
    const Circuit round = parse_circuit(render_circuit(qft));
    REQUIRE(round.num_qubits == 10 && round.gates == qft.gates);
    threw = false;
    try {
        parse_circuit("qubits 3\nh 7\n");
    } catch (const ParseError &e) {
        threw = e.line() == 2;
    }
    REQUIRE(threw);
    // dense reference: QFT|k> is the DFT column
    const int n = 10;
    const uint64_t k = 291;
    DenseState ds = ref_run(qft, make_dense_basis(n, k));
    const double N = 1 << n;
    for (uint64_t j = 0; j < (1u << n); j += 37) {
        const double ang = 2.0 * std::numbers::pi * (double)((k * j) % (1u << n)) / N;
        REQUIRE(std::abs(ds.amps[j] - std::polar(1.0 / std::sqrt(N), ang)) < 1e-10);
    }
    // GPU engine: QFT-10 on |k>, slices of 2^6; fidelity vs the dense run
    EngineConfig ec;
    ec.slice_bits = 6;
    ec.codec = CodecConfig{CodecMode::Absolute, 1e-5, 16, Predictor::PreviousValue};
    auto [eng, m] = run(qft, ec, init_basis_state(n, k, 6));
    REQUIRE(m.gates == qft.gate_count());
    REQUIRE(m.min_compression_ratio > 0.0 && m.dense_bytes == (16u << n));
    const StateVector out = eng->gather_state();
    const StateVector ref = state_from_amplitudes(n, ds.amps, 6);
    const double f = fidelity(out, ref);
    REQUIRE(f > 0.999);
    const auto slices = eng->compressed_slices();
    REQUIRE(slices.size() == (1u << (n - 6)));
    std::stringstream dump;
    write_state_dump(out, dump);
    const StateVector rd = read_state_dump(dump, 6);
    REQUIRE(std::fabs(fidelity(rd, out) - global_sq_norm(out) * global_sq_norm(out)) < 1e-9);
    // per-gate metrics, overhead factor and the report
    REQUIRE(m.per_gate_min_ratio.size() == qft.gate_count());
    double pmin = 1e300;
    for (double r : m.per_gate_min_ratio) pmin = std::min(pmin, r);
    REQUIRE(pmin >= m.min_compression_ratio);
    const auto rows = eng->gate_metrics();
    REQUIRE(rows.size() == qft.gate_count() + 1 && rows[0].gate_index == -1);
    REQUIRE(rows.back().compressed_bytes > 0);
    const RunMetrics mo = measure_overhead(qft, ec, init_basis_state(n, k, 6));
    REQUIRE(mo.baseline_wall_seconds > 0.0 && mo.overhead_factor > 0.0);
    const std::string js = metrics_json(mo, rows), csv = metrics_csv(rows);
    REQUIRE(js.find("\"overhead_factor\"") != std::string::npos && js.find("\"per_gate\"") != std::string::npos);
    REQUIRE(csv.rfind("gate_index,min_ratio,mean_ratio,seconds\n", 0) == 0);
    // checkpoint -> resume: the resumed engine holds the same
    // blocks and continues identically
    {
        Engine again(n, ec);
        again.resume(slices, eng->slice_norms(), qft.gate_count());
        const auto s2 = again.compressed_slices();
        REQUIRE(s2.size() == slices.size());
        for (size_t j = 0; j < slices.size(); ++j)
            REQUIRE(s2[j].re.to_bytes() == slices[j].re.to_bytes() && s2[j].im.to_bytes() == slices[j].im.to_bytes());
        const std::vector<GateAction> more{gate_action(Gate::h(3)), gate_action(Gate::h(9))};
        again.run(more);
        eng->run(more);
        const auto a1 = eng->compressed_slices(), a2 = again.compressed_slices();
        for (size_t j = 0; j < a1.size(); ++j)
            REQUIRE(a1[j].re.to_bytes() == a2[j].re.to_bytes() && a1[j].im.to_bytes() == a2[j].im.to_bytes());
    }
    std::printf("api_smoke ok: fidelity %.9f, min ratio %.3f, overhead %.2fx\n", f, m.min_compression_ratio,
                mo.overhead_factor);
    return 0;
}
