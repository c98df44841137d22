// EMG1 operator snapshots through the B200 drop-in (include/emie/greens.hpp):
// the checks of test_greens.cpp:289-348 (round trip bit-for-bit, foreign files
// rejected) on an operator built on the device, plus a checksum line the GPU
// test compares with the reference's own load_operator reading the same file
// (oracle/ref_tool.cpp snapshot-check). Usage: dropin_snapshot <dir>
#include <cmath>
#include <complex>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "emie/greens.hpp"

namespace fs = std::filesystem;

static int fails = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s (line %d)\n", #c, __LINE__); \
      ++fails;                                                     \
    }                                                              \
  } while (0)

static double checksum(const emie::CompressedGreensOperator& op) {
  double s = 0.0;
  double w = 1.0;
  for (const auto& b : op.blocks)
    for (const auto* c : {&b.xx, &b.yy, &b.zz, &b.xy, &b.xz, &b.yz})
      for (const auto& v : *c) {
        s += w * (v.real() + 0.5 * v.imag());
        w = w * 1.000001 + 1e-3;
      }
  return s;
}

int main(int argc, char** argv) {
  const fs::path dir = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path();
  emie::LayeredModel m;
  m.tops = {0.0, 400.0};
  m.sigma = {0.0, 0.02, 0.5};
  const double omega = 2.0 * 3.141592653589793 / 10.0;
  emie::AnomalyGrid grid = emie::make_grid(m, {0.0, 150.0, 300.0}, 3, 2, 200.0, 260.0, 0.0, 0.0);
  const emie::CompressedGreensOperator op = emie::assemble_operator(grid, m, omega);

  const fs::path good = dir / "emie_b200_snapshot.bin", bad = dir / "emie_b200_snapshot_bad.bin";
  emie::save_operator(good.string(), op);
  const auto re = emie::load_operator(good.string());
  EXPECT(re.has_value());
  if (re) {
    EXPECT(re->nx == op.nx && re->ny == op.ny && re->nz == op.nz && re->omega == op.omega);
    EXPECT(re->blocks.size() == op.blocks.size());
    for (std::size_t i = 0; i < op.blocks.size() && i < re->blocks.size(); ++i) {
      EXPECT(re->blocks[i].xx == op.blocks[i].xx);
      EXPECT(re->blocks[i].yy == op.blocks[i].yy);
      EXPECT(re->blocks[i].zz == op.blocks[i].zz);
      EXPECT(re->blocks[i].xy == op.blocks[i].xy);
      EXPECT(re->blocks[i].xz == op.blocks[i].xz);
      EXPECT(re->blocks[i].yz == op.blocks[i].yz);
    }
  }
  std::vector<char> bytes;
  {
    std::ifstream is(good, std::ios::binary);
    bytes.assign(std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>());
  }
  EXPECT(bytes.size() > 16);
  {
    std::vector<char> mod = bytes;
    mod[0] ^= 0x5a;
    std::ofstream os(bad, std::ios::binary | std::ios::trunc);
    os.write(mod.data(), static_cast<std::streamsize>(mod.size()));
  }
  EXPECT(!emie::load_operator(bad.string()).has_value());
  {
    std::ofstream os(bad, std::ios::binary | std::ios::trunc);
    os.write(bytes.data(), static_cast<std::streamsize>(bytes.size() / 2));
  }
  EXPECT(!emie::load_operator(bad.string()).has_value());
  EXPECT(!emie::load_operator((dir / "emie_b200_absent.bin").string()).has_value());
  fs::remove(bad);
  std::printf("{\"path\": \"%s\", \"nx\": %d, \"ny\": %d, \"nz\": %d, \"omega\": %.17g, \"bytes\": %zu, "
              "\"checksum\": %.17g, \"failures\": %d}\n",
              good.string().c_str(), op.nx, op.ny, op.nz, op.omega, bytes.size(), checksum(op), fails);
  return fails == 0 ? 0 : 1;
}
