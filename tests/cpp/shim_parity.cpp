// Reference-style parity test re-pointed at the C++ shim (include/pcpq_gpu.hpp):
// the shape of proj/tests/test_pq_index.cpp's scoring checks, against golden
// vectors produced by the unmodified reference library.
//
//   shim_parity <index.idx> <queries.f32> <B> <scores.f32> <ids10.i32> <top10.f32> <eta0.f32>
// Exit 0 iff score_query / build_lookup_table / score_all / search agree bit-for-bit.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <vector>

#include "pcpq_gpu.hpp"

template <class T>
static std::vector<T> slurp(const char* path) {
  std::ifstream in(path, std::ios::binary);
  std::vector<char> b((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::vector<T> v(b.size() / sizeof(T));
  std::memcpy(v.data(), b.data(), v.size() * sizeof(T));
  return v;
}

int main(int argc, char** argv) {
  if (argc != 8) return 2;
  const auto bytes = slurp<std::uint8_t>(argv[1]);
  const auto Q = slurp<float>(argv[2]);
  const std::uint32_t B = static_cast<std::uint32_t>(std::atoi(argv[3]));
  const auto scores = slurp<float>(argv[4]);
  const auto ids10 = slurp<std::int32_t>(argv[5]);
  const auto top10 = slurp<float>(argv[6]);
  const auto eta0 = slurp<float>(argv[7]);
  int bad = 0;
  try {
    const pcpq::gpu::Index idx = pcpq::gpu::deserialize(bytes, 0);
    const std::size_t n = idx.n(), d = idx.d();
    for (std::uint32_t b = 0; b < B; ++b) {
      const std::span<const float> q(Q.data() + b * d, d);
      const auto s = pcpq::gpu::score_query(idx, q);
      if (std::memcmp(s.data(), scores.data() + b * n, n * 4) != 0) ++bad;
    }
    pcpq::gpu::ScoreCounters c;
    const auto lut = pcpq::gpu::build_lookup_table(idx, std::span<const float>(Q.data(), d), &c);
    if (std::memcmp(lut.eta.data(), eta0.data(), eta0.size() * 4) != 0) ++bad;
    const auto s0 = pcpq::gpu::score_all(idx, lut, &c);
    if (std::memcmp(s0.data(), scores.data(), n * 4) != 0) ++bad;
    if (c.lookups != n * idx.m() || c.adds != n * (idx.m() - 1)) ++bad;
    const auto r = pcpq::gpu::search(idx, Q, B, 10);
    if (std::memcmp(r.ids.data(), ids10.data(), ids10.size() * 4) != 0) ++bad;
    if (std::memcmp(r.scores.data(), top10.data(), top10.size() * 4) != 0) ++bad;
    // the same index sharded over two "devices" of this process (the one GPU twice,
    // peer-copy transport): the merged top-n equals the unsharded one
    if (n >= 2) {
      const int devs[2] = {0, 0};
      const pcpq::gpu::MultiIndex mx(bytes, devs, PCPQG_TRANSPORT_PEER);
      if (mx.n() != n || mx.devices() != 2) ++bad;
      const auto rm = mx.search(Q, B, 10);
      if (std::memcmp(rm.ids.data(), ids10.data(), ids10.size() * 4) != 0) ++bad;
      if (std::memcmp(rm.scores.data(), top10.data(), top10.size() * 4) != 0) ++bad;
    }
    // error taxonomy through the shim: a wrong query width is size_mismatch
    try {
      std::vector<float> q2(d + 1, 0.0f);
      pcpq::gpu::score_query(idx, q2);
      ++bad;
    } catch (const pcpq::gpu::error& e) {
      if (e.code() != pcpq::gpu::errc::size_mismatch) ++bad;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 3;
  }
  std::printf("%s\n", bad ? "FAIL" : "OK");
  return bad ? 1 : 0;
}
