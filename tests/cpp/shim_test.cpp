// C++ parity test through include/multiverse_b200.hpp — written the way the reference's own
// tests would drive multiverse::dag / multiverse::kv (tests/oracles.hpp, SPEC.md known answers).
// Built by tests/test_cpp_shim.py; runs on a GPU box (the device store needs a GPU).
#include <cstdio>
#include <cstdlib>
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

  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("shim ok\n");
  return 0;
}
