// PGM I/O of the C++ drop-in (include/dctfilter_b200.hpp), host only: the
// reference's PgmTest cases (image_test.cc:36-77). Run by tests/test_pgm.py.
#include <cstdio>

#include "dctfilter_b200.hpp"

using namespace dctfilter_b200;

static int failures = 0;
#define CHECK(c, what)                                   \
  do {                                                   \
    const bool ok_ = (c);                                \
    std::printf("[%s] %s\n", ok_ ? "PASS" : "FAIL", what); \
    if (!ok_) ++failures;                                \
  } while (0)

template <class F>
bool throws_pgm(F f) {
  try {
    f();
  } catch (const PgmError&) {
    return true;
  }
  return false;
}

int main() {
  const std::string p5 = std::string("P5\n2 2\n255\n") + std::string("\x00\xff\x11\x22", 4);
  const GrayImage a = load_pgm(p5);
  CHECK(a.width == 2 && a.height == 2 && a.samples == std::vector<std::uint8_t>({0x00, 0xff, 0x11, 0x22}),
        "parses minimal P5");
  const GrayImage b = load_pgm(std::string("P2\n# a comment\n2 2\n255\n0 255\n17 34\n"));
  CHECK(b.samples == a.samples, "P2 and P5 agree");
  GrayImage r{37, 21, std::vector<std::uint8_t>(37 * 21)};
  for (size_t i = 0; i < r.samples.size(); ++i) r.samples[i] = std::uint8_t(i * 37 + 11);
  const GrayImage back = load_pgm(save_pgm(r));
  CHECK(back.width == 37 && back.height == 21 && back.samples == r.samples, "save/load round trip");
  CHECK(throws_pgm([] { load_pgm(std::string("P6\n2 2\n255\n")); }), "rejects P6");
  CHECK(throws_pgm([] { load_pgm(std::string("P5\n2 2\n511\n")); }), "rejects maxval 511");
  CHECK(throws_pgm([] { load_pgm(std::string("P5\n-2 2\n255\n")); }), "rejects negative size");
  CHECK(throws_pgm([] { load_pgm(std::string("P5\nx 2\n255\n")); }), "rejects non-integer");
  CHECK(throws_pgm([] { load_pgm(std::string("P5\n2 2\n255\nab")); }), "rejects truncated P5");
  CHECK(throws_pgm([] { load_pgm(std::string("P2\n2 2\n255\n0 1 2")); }), "rejects truncated P2");
  CHECK(throws_pgm([] { load_pgm_file("/nonexistent/x.pgm"); }), "missing file");
  std::printf("%s\n", failures ? "FAILED" : "ALL PASSED");
  return failures ? 1 : 0;
}
