// qcsim/codec.hpp -- QCB1 error-bounded codec, B200 implementation.
//
// Same declarations as /root/reference/proj/include/qcsim/codec.hpp:41-108
// (enum values, field order and defaults, constants, signatures).
// compress_plane / decompress_plane run on the GPU through the C-ABI
// (qcsim_compress_plane / qcsim_decompress_plane) and produce byte-identical
// blocks and bit-identical values.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <utility>
#include <vector>

namespace qcsim {

enum class CodecMode : uint8_t { RangeRelative = 0, Absolute = 1, Lossless = 2 };
enum class Predictor : uint8_t { PreviousValue = 0, LinearExtrapolation = 1 };

struct CodecConfig {
    CodecMode mode = CodecMode::RangeRelative;
    double bound = 0.01;
    int quant_code_bits = 16; // [4, 24]
    Predictor predictor = Predictor::PreviousValue;

    void validate() const; // std::invalid_argument
};

struct CompressedBlock {
    CodecMode mode = CodecMode::RangeRelative;
    Predictor predictor = Predictor::PreviousValue;
    uint8_t quant_code_bits = 16;
    uint64_t element_count = 0;
    double effective_abs_bound = 0.0;
    uint64_t outlier_count = 0;
    std::vector<uint8_t> payload;

    static constexpr size_t kHeaderBytes = 40;
    static constexpr uint8_t kFormatVersion = 1;

    uint64_t byte_size() const { return kHeaderBytes + payload.size(); }
    void append_bytes(std::vector<uint8_t> &out) const;
    std::vector<uint8_t> to_bytes() const;
    static CompressedBlock from_bytes(std::span<const uint8_t> bytes, size_t *consumed = nullptr);
};

struct CodecStats {
    uint64_t input_bytes = 0;
    uint64_t output_bytes = 0;
    double ratio = 0.0;
    double outlier_fraction = 0.0;
};

std::pair<CompressedBlock, CodecStats> compress_plane(std::span<const double> values, const CodecConfig &config);
std::vector<double> decompress_plane(const CompressedBlock &block);

inline double compression_ratio(const CodecStats &stats) {
    return static_cast<double>(stats.input_bytes) / static_cast<double>(stats.output_bytes);
}

} // namespace qcsim
