// RMAT synthetic edge streams — host utility used to
// prepare benchmark inputs; bit-identical to synth.py's NumPy generator.
//
// Candidate i draws `scale` quadrant choices from a counter-based stream:
// word j of candidate i is splitmix64(base + 16*i + j/2), 32 bits per level
// (low half first), base = seed_for(seed, 0x3A7).  Self-loops are dropped; the
// FIRST occurrence (smallest i) of every unordered pair is kept, in candidate
// order, until num_edges pairs exist; ids are compacted to 0..|V|-1 by rank.
#include <parallel/algorithm>

#include <algorithm>
#include <cstring>
#include <vector>

#include "artifact.hpp"

using namespace catgnn;

namespace {

struct Cand {
  uint64_t key;  // (min << 32) | max, or ~0 for self-loops
  uint64_t idx;
  bool operator<(const Cand& o) const { return key != o.key ? key < o.key : idx < o.idx; }
};

inline void draw(uint64_t base, uint64_t i, int scale, uint32_t ta, uint32_t tab, uint32_t tabc,
                 uint64_t* src, uint64_t* dst) {
  uint64_t s = 0, d = 0, word = 0;
  for (int l = 0; l < scale; ++l) {
    if ((l & 1) == 0) word = mix64(base + 16 * i + (uint64_t)(l >> 1));
    const uint32_t r = (l & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
    const uint64_t bs = r >= tab;
    const uint64_t bd = (r >= ta && r < tab) || r >= tabc;
    s |= bs << (scale - 1 - l);
    d |= bd << (scale - 1 - l);
  }
  *src = s;
  *dst = d;
}

}  // namespace

extern "C" int catgnn_synth_rmat(uint32_t scale, uint64_t num_edges, double a, double b, double c,
                                 uint64_t seed, uint64_t* out_edges, uint64_t* num_nodes) {
  return guarded([&] {
    if (scale < 1 || scale > 32) throw ConfigError("rmat scale must be in [1, 32]");
    if (!out_edges || !num_nodes) throw ConfigError("null output");
    const uint64_t base = seed_for(seed, 0x3A7);
    auto thr = [](double p) { return (uint32_t)std::min(p * 4294967296.0, 4294967295.0); };
    const uint32_t ta = thr(a), tab = thr(a + b), tabc = thr(a + b + c);
    uint64_t n_cand = num_edges + num_edges * 3 / 10 + 1024;
    std::vector<uint64_t> chosen;
    for (int attempt = 0; attempt < 16; ++attempt) {
      std::vector<Cand> cand(n_cand);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < (int64_t)n_cand; ++i) {
        uint64_t s, d;
        draw(base, (uint64_t)i, (int)scale, ta, tab, tabc, &s, &d);
        cand[i].idx = (uint64_t)i;
        cand[i].key = s == d ? ~0ull : ((std::min(s, d) << 32) | std::max(s, d));
      }
      __gnu_parallel::sort(cand.begin(), cand.end());
      chosen.clear();
      for (uint64_t i = 0; i < n_cand; ++i) {
        if (cand[i].key == ~0ull) break;
        if (i == 0 || cand[i].key != cand[i - 1].key) chosen.push_back(cand[i].idx);
      }
      if (chosen.size() >= num_edges) break;
      n_cand = n_cand + n_cand / 2;
    }
    if (chosen.size() < num_edges) throw ConfigError("more edges requested than the RMAT graph can supply");
    __gnu_parallel::sort(chosen.begin(), chosen.end());
    chosen.resize(num_edges);
    const uint64_t ids = 1ull << scale;
    std::vector<uint8_t> seen(ids, 0);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)num_edges; ++k) {
      uint64_t s, d;
      draw(base, chosen[k], (int)scale, ta, tab, tabc, &s, &d);
      out_edges[2 * k] = s;
      out_edges[2 * k + 1] = d;
      seen[s] = 1;  // benign races: every writer stores 1
      seen[d] = 1;
    }
    std::vector<uint64_t> rank(ids);
    uint64_t r = 0;
    for (uint64_t v = 0; v < ids; ++v) {
      rank[v] = r;
      r += seen[v];
    }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)(2 * num_edges); ++k) out_edges[k] = rank[out_edges[k]];
    *num_nodes = r;
  });
}
