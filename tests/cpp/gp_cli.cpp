// gp_cli.cpp — C++ host program over include/gradpack_b200.hpp (the drop-in a
// gradpack C++ caller would use).  Driven by tests/test_gpu_cpp.py:
//   gp_cli encode <grad.f32> <r> <index> <value> <fpr> <seed> <out.drc>
//   gp_cli decode <in.drc> <out.support.u32> <out.values.f64>
// Exit code 0 on success; 10 + gp_status for a gradpack_b200::Error (the
// exception class the reference would have thrown, errors.hpp:21-53).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/gradpack_b200.hpp"

namespace gb = gradpack_b200;

static std::vector<uint8_t> slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  return std::vector<uint8_t>(std::istreambuf_iterator<char>(f), {});
}

static void spit(const char* path, const void* p, size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
}

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "encode" && argc == 9) {
      const std::vector<uint8_t> raw = slurp(argv[2]);
      const uint64_t d = raw.size() / 4;
      gb::PipelineConfig cfg = gb::default_config();
      cfg.index_method = static_cast<uint8_t>(std::atoi(argv[4]));
      cfg.value_method = static_cast<uint8_t>(std::atoi(argv[5]));
      cfg.fpr = std::atof(argv[6]);
      cfg.seed = std::strtoull(argv[7], nullptr, 10);
      gb::Context ctx(d);
      const auto c = gb::compress_dense(ctx, reinterpret_cast<const float*>(raw.data()), d,
                                        std::strtoull(argv[3], nullptr, 10), cfg);
      const gp_volume_report v = gb::volume(c);
      std::printf("bytes=%zu total_bits=%llu index_bits=%llu value_bits=%llu\n", c.size(),
                  static_cast<unsigned long long>(v.total_bits), static_cast<unsigned long long>(v.index_bits),
                  static_cast<unsigned long long>(v.value_bits));
      spit(argv[8], c.data(), c.size());
      return 0;
    }
    if (cmd == "decode" && argc == 5) {
      const std::vector<uint8_t> c = slurp(argv[2]);
      gb::Context ctx(1 << 22);
      const gb::SparseGradient sg = gb::decompress_gradient(ctx, c, 1 << 22);
      spit(argv[3], sg.support.data(), sg.support.size() * 4);
      spit(argv[4], sg.values.data(), sg.values.size() * 8);
      std::printf("dim=%llu count=%zu\n", static_cast<unsigned long long>(sg.dim), sg.support.size());
      return 0;
    }
    std::fprintf(stderr, "usage: gp_cli encode|decode ...\n");
    return 2;
  } catch (const gb::TruncatedError& e) {
    std::fprintf(stderr, "TruncatedError: %s\n", e.what());
    return 10 + GP_TRUNCATED;
  } catch (const gb::ChecksumError& e) {
    std::fprintf(stderr, "ChecksumError: %s\n", e.what());
    return 10 + GP_CHECKSUM;
  } catch (const gb::UnknownMethodError& e) {
    std::fprintf(stderr, "UnknownMethodError: %s\n", e.what());
    return 10 + GP_UNKNOWN_METHOD;
  } catch (const gb::CorruptPayloadError& e) {
    std::fprintf(stderr, "CorruptPayloadError: %s\n", e.what());
    return 10 + GP_CORRUPT_PAYLOAD;
  } catch (const gb::DecodeError& e) {
    std::fprintf(stderr, "DecodeError: %s\n", e.what());
    return 10 + GP_DECODE;
  } catch (const gb::Error& e) {
    std::fprintf(stderr, "Error: %s\n", e.what());
    return 10 + GP_ERROR;
  }
}
