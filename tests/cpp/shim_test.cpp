// C++ parity test through include/multiverse_b200.hpp — written the way the reference's own
// tests would drive multiverse::dag / multiverse::kv (tests/oracles.hpp, SPEC.md known answers).
// Built by tests/test_cpp_shim.py; runs on a GPU box (the device store needs a GPU).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "multiverse_b200.hpp"

namespace mvb = multiverse_b200;

static int failures = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #c); \
      ++failures;                                                   \
    }                                                               \
  } while (0)

// ---- attention through the shim: attn::prefill over T1 and attn::decode of two forked branches, against
// an fp64 restatement of toy_model.cpp:121-157 (interleaved RoPE :30-41, scores / sqrt(128), self last) ----
static float bf16_round(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  std::memcpy(&x, &u, 4);
  return x;
}
static uint16_t bf16_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return (uint16_t)(u >> 16);
}
static std::vector<double> rope(const std::vector<double>& x, int rows, int heads, const std::vector<int>& pos) {
  std::vector<double> y = x;
  for (int r = 0; r < rows; ++r)
    for (int h = 0; h < heads; ++h)
      for (int t = 0; t < 64; ++t) {
        const double th = pos[r] * std::pow(10000.0, -2.0 * t / 128.0), c = std::cos(th), s = std::sin(th);
        double* v = y.data() + ((size_t)r * heads + h) * 128 + 2 * t;
        const double a = v[0], b = v[1];
        v[0] = a * c - b * s;
        v[1] = a * s + b * c;
      }
  return y;
}
// one query row (heads hq) over context rows `ctx` (self last): fp64
static void attend(const double* q, const std::vector<double>& K, const std::vector<double>& V, int hq, int hkv,
                   const std::vector<int>& ctx, double* out) {
  for (int h = 0; h < hq; ++h) {
    const int kvh = h / (hq / hkv);
    std::vector<double> sc;
    double mx = -1e300;
    for (int j : ctx) {
      double s = 0;
      for (int d = 0; d < 128; ++d) s += q[h * 128 + d] * K[((size_t)j * hkv + kvh) * 128 + d];
      sc.push_back(s / std::sqrt(128.0));
      mx = std::max(mx, sc.back());
    }
    double den = 0;
    for (auto& s : sc) den += (s = std::exp(s - mx));
    for (int d = 0; d < 128; ++d) {
      double acc = 0;
      for (size_t k = 0; k < ctx.size(); ++k) acc += sc[k] * V[((size_t)ctx[k] * hkv + kvh) * 128 + d];
      out[h * 128 + d] = acc / den;
    }
  }
}

static void attention_parity(const std::vector<int32_t>& t1, const mvb::dag::VisibilitySpec& spec) {
  const int n = (int)t1.size(), hq = 8, hkv = 2;
  uint64_t seed = 12345;
  auto rnd = [&]() {
    seed = seed * 6364136223846793005ULL + 1442695040888963407ULL;
    return bf16_round((float)((double)(seed >> 11) * 0x1.0p-53 * 2.0 - 1.0));
  };
  std::vector<float> q(n * hq * 128), k(n * hkv * 128), v(n * hkv * 128);
  for (auto& x : q) x = rnd();
  for (auto& x : k) x = rnd();
  for (auto& x : v) x = rnd();
  auto to_dev = [](const std::vector<float>& h) {
    std::vector<uint16_t> b(h.size());
    for (size_t i = 0; i < h.size(); ++i) b[i] = bf16_bits(h[i]);
    mvb::DeviceBuffer<uint16_t> d(h.size());
    d.upload(b.data(), b.size());
    return d;
  };
  const std::vector<double> q64(q.begin(), q.end()), k64(k.begin(), k.end()), v64(v.begin(), v.end());
  const std::vector<double> Kr = rope(k64, n, hkv, spec.positions);
  const std::vector<double> Qr = rope(q64, n, hq, spec.positions);
  double worst = 0;

  // prefill: every row over its mask-visible rows, then self (toy_model.cpp:183-196)
  auto vis = mvb::dag::build_visibility_device(t1);
  auto dq = to_dev(q), dk = to_dev(k), dv = to_dev(v);
  mvb::DeviceBuffer<float> out(n * hq * 128);
  mvb::attn::prefill(dq.data(), dk.data(), dv.data(), vis, hq, hkv, out.data(), true);
  mvb::cuda_check(cudaDeviceSynchronize());
  auto got = out.download();
  for (int i = 0; i < n; ++i) {
    std::vector<int> ctx;
    for (int j = 0; j < i; ++j)
      if (spec.mask.at(i, j)) ctx.push_back(j);
    ctx.push_back(i);
    std::vector<double> ref(hq * 128);
    attend(Qr.data() + (size_t)i * hq * 128, Kr, v64, hq, hkv, ctx, ref.data());
    for (int e = 0; e < hq * 128; ++e) worst = std::max(worst, std::abs(ref[e] - got[(size_t)i * hq * 128 + e]));
  }
  EXPECT(worst < 2e-3);

  // decode: a 12-token prefix appended one token at a time, forked into 2 branches of 1 new token each
  // (positions 12, the shared start), both decoded in one launch
  mvb::kv::RadixStore st(0, 4096, /*layers=*/1, /*kv_heads=*/hkv);
  auto root = st.create();
  mvb::DeviceBuffer<int32_t> d_tok(1), d_pos(2);
  for (int t = 0; t < 12; ++t) {
    mvb::DeviceBuffer<uint16_t> kt(hkv * 128), vt(hkv * 128);
    std::vector<uint16_t> kb(hkv * 128), vb(hkv * 128);
    for (int e = 0; e < hkv * 128; ++e) kb[e] = bf16_bits(k[t * hkv * 128 + e]), vb[e] = bf16_bits(v[t * hkv * 128 + e]);
    kt.upload(kb.data(), kb.size());
    vt.upload(vb.data(), vb.size());
    const int32_t tp[2] = {t1[t], t};
    mvb::DeviceBuffer<int32_t> io(2);
    io.upload(tp, 2);
    const std::uint64_t h = root.id;
    st.append(std::span<const std::uint64_t>(&h, 1), io.data(), io.data() + 1, 0, kt.data(), vt.data());
  }
  root.length = 12;
  auto br = st.fork(root, 2);
  const std::uint64_t hs[2] = {br[0].id, br[1].id};
  // rows 12 (branch 0's token) and 17 (branch 1's): k, v, q rows of T1, both at position 12
  const int rows[2] = {12, 17};
  std::vector<uint16_t> kb(2 * hkv * 128), vb(2 * hkv * 128), qb(2 * hq * 128);
  for (int b = 0; b < 2; ++b) {
    for (int e = 0; e < hkv * 128; ++e) kb[b * hkv * 128 + e] = bf16_bits(k[rows[b] * hkv * 128 + e]);
    for (int e = 0; e < hkv * 128; ++e) vb[b * hkv * 128 + e] = bf16_bits(v[rows[b] * hkv * 128 + e]);
    for (int e = 0; e < hq * 128; ++e) qb[b * hq * 128 + e] = bf16_bits(q[rows[b] * hq * 128 + e]);
  }
  mvb::DeviceBuffer<uint16_t> dk2(kb.size()), dv2(vb.size()), dq2(qb.size());
  dk2.upload(kb.data(), kb.size());
  dv2.upload(vb.data(), vb.size());
  dq2.upload(qb.data(), qb.size());
  const int32_t tp[4] = {t1[12], t1[17], 12, 12};
  mvb::DeviceBuffer<int32_t> io(4);
  io.upload(tp, 4);
  st.append(std::span<const std::uint64_t>(hs, 2), io.data(), io.data() + 2, 0, dk2.data(), dv2.data());
  mvb::DeviceBuffer<float> dout(2 * hq * 128);
  mvb::attn::decode(st, 0, std::span<const std::uint64_t>(hs, 2), hq, dq2.data(), io.data() + 2, dout.data(), true);
  mvb::cuda_check(cudaDeviceSynchronize());
  auto dgot = dout.download();
  // the host reference: keys rotated at their positions (0..11, then 12), the query at 12
  double dworst = 0;
  for (int b = 0; b < 2; ++b) {
    std::vector<double> K2, V2;
    std::vector<int> pos;
    for (int t = 0; t < 12; ++t) pos.push_back(t);
    pos.push_back(12);
    std::vector<double> kk, vv;
    for (int t = 0; t < 12; ++t)
      for (int e = 0; e < hkv * 128; ++e) kk.push_back(k64[t * hkv * 128 + e]), vv.push_back(v64[t * hkv * 128 + e]);
    for (int e = 0; e < hkv * 128; ++e) kk.push_back(k64[rows[b] * hkv * 128 + e]), vv.push_back(v64[rows[b] * hkv * 128 + e]);
    const std::vector<double> Kb = rope(kk, 13, hkv, pos);
    std::vector<double> qq(q64.begin() + rows[b] * hq * 128, q64.begin() + (rows[b] + 1) * hq * 128);
    const std::vector<double> Qb = rope(qq, 1, hq, std::vector<int>{12});
    std::vector<int> ctx;
    for (int t = 0; t <= 12; ++t) ctx.push_back(t);
    std::vector<double> ref(hq * 128);
    attend(Qb.data(), Kb, vv, hq, hkv, ctx, ref.data());
    for (int e = 0; e < hq * 128; ++e) dworst = std::max(dworst, std::abs(ref[e] - dgot[(size_t)b * hq * 128 + e]));
  }
  EXPECT(dworst < 2e-3);
  std::printf("attention: prefill max-abs %.3e, decode max-abs %.3e (tolerance 2e-3)\n", worst, dworst);
}

int main() {
  // SPEC.md:143-160 T1 (data/fixtures/t1.txt == tests/oracles.hpp:42-45) as tokenizer ids.
  const std::vector<int32_t> t1 = {10, 0, 2, 4, 11, 12, 5, 4, 13, 14, 5, 3, 6, 11, 15, 16, 7, 6, 13, 17, 18, 19, 7, 8, 20, 9, 1, 21};
  auto spec = mvb::dag::build_visibility(t1);
  // positions 0..11 | 12..16 | 12..17 | 18..21 | 22
  std::vector<int> want;
  for (int p = 0; p <= 11; ++p) want.push_back(p);
  for (int p = 12; p <= 16; ++p) want.push_back(p);
  for (int p = 12; p <= 17; ++p) want.push_back(p);
  for (int p = 18; p <= 22; ++p) want.push_back(p);
  EXPECT(spec.positions == want);
  // rows 17-22 (path 2) exclude columns 12-16 (path 1); rows >= 23 see every earlier row
  for (std::size_t i = 0; i < t1.size(); ++i)
    for (std::size_t j = 0; j < t1.size(); ++j) {
      bool vis = j <= i && !(i >= 17 && i <= 22 && j >= 12 && j <= 16);
      EXPECT(spec.mask.at(i, j) == vis);
    }

  // grammar::ParseError on a malformed stream (</Parallel> without an open block)
  bool threw = false;
  try {
    mvb::dag::build_visibility(std::vector<int32_t>{10, 1});
  } catch (const mvb::grammar::ParseError& e) {
    threw = e.kind() == mvb::grammar::ParseError::Kind::MalformedStructure;
  }
  EXPECT(threw);

  // kv: SPEC.md:252 zero-copy merge — prefix 12 tokens, paths of 5 and 6, merged length 23
  mvb::kv::RadixStore store(8, 4096);
  auto root = store.create();
  std::vector<int32_t> pre(t1.begin(), t1.begin() + 12);
  std::vector<std::byte> pl(pre.size() * 8, std::byte{7});
  auto prefix = store.extend(root, pre, pl);
  EXPECT(prefix.length == 12);
  auto kids = store.fork(prefix, 2);
  EXPECT(kids.size() == 2 && kids[0].length == 12);
  auto a = store.extend(kids[0], std::vector<int32_t>(t1.begin() + 12, t1.begin() + 17));
  auto b = store.extend(kids[1], std::vector<int32_t>(t1.begin() + 17, t1.begin() + 23));
  std::vector<mvb::kv::SequenceHandle> br = {a, b};
  auto merged = store.merge(prefix, br);
  EXPECT(merged.length == 23);
  EXPECT(store.stats().bytes_copied_on_last_op == 0);
  auto toks = store.resolve(merged);
  EXPECT(std::vector<int32_t>(toks.begin(), toks.end()) == std::vector<int32_t>(t1.begin(), t1.begin() + 23));
  auto sp = store.resolve_slots(prefix), sm = store.resolve_slots(merged), sa = store.resolve_slots(a);
  for (int i = 0; i < 12; ++i) EXPECT(sp[i] == sm[i]);             // prefix shared, not copied
  for (int i = 0; i < 5; ++i) EXPECT(sa[12 + i] == sm[12 + i]);     // branch suffix shared
  auto pay = store.resolve_payloads(merged);
  EXPECT(pay.size() == 23 * 8 && pay[0] == std::byte{7});

  // CacheError kinds (kvcache.hpp:32-41)
  store.release(a);
  threw = false;
  try {
    store.release(a);
  } catch (const mvb::kv::CacheError& e) {
    threw = e.kind() == mvb::kv::CacheError::Kind::DoubleRelease;
  }
  EXPECT(threw);
  threw = false;
  try {
    auto other = store.create();
    auto o2 = store.extend(other, std::vector<int32_t>{1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13});
    std::vector<mvb::kv::SequenceHandle> bad = {o2};
    store.merge(prefix, bad);
  } catch (const mvb::kv::CacheError& e) {
    threw = e.kind() == mvb::kv::CacheError::Kind::BranchNotDescendant;
  }
  EXPECT(threw);
  threw = false;
  try {
    mvb::kv::RadixStore tiny(0, 32);
    auto h = tiny.create();
    tiny.extend(h, std::vector<int32_t>(64, 11));
  } catch (const mvb::kv::CacheError& e) {
    threw = e.kind() == mvb::kv::CacheError::Kind::CapacityExceeded;
  }
  EXPECT(threw);

  attention_parity(t1, spec);

  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("shim ok\n");
  return 0;
}
