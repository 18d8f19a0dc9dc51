// Our test (not the reference's): the GPU wrappers of prefixopt/b200.hpp
// against the reference's own CPU implementations, which these includes
// resolve to in /root/reference (cost.hpp: dedup, cache_sim.hpp: simulate).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <random>
#include <string>
#include <vector>

#include "prefixopt/b200.hpp"
#include "prefixopt/cache_sim.hpp"
#include "prefixopt/cost.hpp"

using namespace prefixopt;

namespace {
std::vector<std::string> random_prompts(std::mt19937& rng, int n) {
  const std::string alpha = "ab \n\t\"x";
  std::vector<std::string> base;
  for (int i = 0; i < 6; ++i) {
    std::string s;
    for (int k = 0, L = int(rng() % 30); k < L; ++k) s += alpha[rng() % alpha.size()];
    base.push_back(s);
  }
  std::vector<std::string> out;
  for (int i = 0; i < n; ++i) {
    std::string s = base[rng() % base.size()];
    s = s.substr(0, rng() % (s.size() + 1));
    for (int k = 0, L = int(rng() % 5); k < L; ++k) s += alpha[rng() % alpha.size()];
    out.push_back(s);
  }
  return out;
}
}  // namespace

TEST_CASE("b200::dedup equals the reference dedup") {
  std::mt19937 rng(1);
  for (int trial = 0; trial < 50; ++trial) {
    auto ps = random_prompts(rng, 1 + int(rng() % 60));
    DedupResult ref = prefixopt::dedup(ps);
    b200::DedupResult got = b200::dedup(ps);
    CHECK(got.uniques == ref.uniques);
    CHECK(got.expansion_map == ref.expansion_map);
  }
}

TEST_CASE("b200::simulate_unbounded equals the reference simulate (eviction none)") {
  std::mt19937 rng(2);
  for (int trial = 0; trial < 50; ++trial) {
    auto ps = random_prompts(rng, 1 + int(rng() % 60));
    for (const Tokenizer* tok : {&char_tokenizer(), &word_tokenizer()}) {
      CacheConfig cfg;
      cfg.min_cacheable_prefix_tokens = rng() % 6;
      SimReport ref = prefixopt::simulate(ps, cfg, *tok);
      b200::ReplayResult got = b200::simulate_unbounded(ps, cfg.min_cacheable_prefix_tokens, *tok);
      REQUIRE(got.input_tokens.size() == ref.requests.size());
      for (size_t i = 0; i < ps.size(); ++i) {
        CHECK(got.input_tokens[i] == ref.requests[i].input_tokens);
        CHECK(got.hit_tokens[i] == ref.requests[i].hit_tokens);
        CHECK(got.miss_tokens[i] == ref.requests[i].miss_tokens);
        CHECK(got.written_tokens[i] == ref.requests[i].written_tokens);
      }
      CHECK(got.total_hit == ref.total_hit);
      CHECK(got.phr == ref.phr);
    }
  }
}

TEST_CASE("b200::render_prompts equals render_prompt per entry") {
  Table t({"title", "q\"t"}, {{"Dune", "a\nb"}, {"It", ""}});
  RequestSchedule s;
  s.entries.push_back({1, {0, 1}});
  s.entries.push_back({0, {1}});
  s.entries.push_back({0, {}});
  auto got = b200::render_prompts(s, t, "SYS", "Q?");
  for (size_t i = 0; i < s.size(); ++i) CHECK(got[i] == render_prompt(s.entries[i], t, "SYS", "Q?"));
}

TEST_CASE("b200::load_csv parses RFC 4180 and reports the reference's errors") {
  Table t = b200::load_csv("a,b\r\n\"x,\"\"y\"\"\",2\n3,\"4\n5\"\n\n");
  REQUIRE(t.row_count() == 2);
  CHECK(t.field_name(1) == "b");
  CHECK(t.cell(0, 0) == "x,\"y\"");
  CHECK(t.cell(1, 1) == "4\n5");
  CHECK_THROWS_AS(b200::load_csv(""), structural_error);
  CHECK_THROWS_AS(b200::load_csv("a,a\n"), schema_error);
  CHECK_THROWS_AS(b200::load_csv("a,b\n1\n"), structural_error);
  CHECK_THROWS_AS(b200::load_csv("a\n\"x"), structural_error);
}
