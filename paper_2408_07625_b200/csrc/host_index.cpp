// Host-side setup for the B200 local-energy path: grouped index, device-layout
// planning. See host_index.h. (The synthetic generators are in synth.cpp.)
#include "host_index.h"

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>

namespace qvmc_b200 {

namespace {

uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

using Words3 = std::array<uint64_t, 3 * kMaxWords>;

struct Words3Hash {
  size_t operator()(const Words3& k) const noexcept {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (uint64_t w : k) {
      h ^= w + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 33;
    }
    return static_cast<size_t>(h);
  }
};

using WordsN = std::array<uint64_t, kMaxWords>;
struct WordsNHash {
  size_t operator()(const WordsN& k) const noexcept { return Words3Hash{}(Words3{k[0], k[1], k[2], k[3]}); }
};

}  // namespace

HostIndex index_from_terms(int n_qubits, int n_words, int64_t n_raw, const double* coeff, const uint64_t* xw,
                           const uint64_t* yw, const uint64_t* zw) {
  if (n_qubits < 1 || n_qubits > 64 * kMaxWords)
    throw std::invalid_argument("HamiltonianIndex: qubit count out of range");
  if (n_words != (n_qubits + 63) / 64) throw std::invalid_argument("HamiltonianIndex: n_words != ceil(N/64)");
  if (n_raw < 0) throw std::invalid_argument("HamiltonianIndex: negative term count");
  const int tail = n_qubits % 64;
  const uint64_t tail_mask = tail ? ((uint64_t{1} << tail) - 1) : ~uint64_t{0};

  // merge duplicate strings, keeping first-occurrence order (hamiltonian.cpp:68-85)
  std::vector<Words3> keys;
  std::vector<double> mcoef;
  std::unordered_map<Words3, size_t, Words3Hash> seen;
  keys.reserve(static_cast<size_t>(n_raw));
  mcoef.reserve(static_cast<size_t>(n_raw));
  seen.reserve(static_cast<size_t>(n_raw) * 2);
  for (int64_t t = 0; t < n_raw; ++t) {
    Words3 k{};
    for (int w = 0; w < n_words; ++w) {
      const uint64_t a = xw[t * n_words + w], b = yw[t * n_words + w], c = zw[t * n_words + w];
      if ((a & b) | (a & c) | (b & c))
        throw std::invalid_argument("HamiltonianIndex: term " + std::to_string(t) + " has overlapping Pauli masks");
      if (w == n_words - 1 && ((a | b | c) & ~tail_mask))
        throw std::invalid_argument("HamiltonianIndex: term " + std::to_string(t) + " has bits beyond the qubit count");
      k[w] = a;
      k[kMaxWords + w] = b;
      k[2 * kMaxWords + w] = c;
    }
    auto [it, fresh] = seen.emplace(k, keys.size());
    if (fresh) {
      keys.push_back(k);
      mcoef.push_back(coeff[t]);
    } else {
      mcoef[it->second] += coeff[t];
    }
  }

  // group survivors by xy = x|y, first-occurrence order (hamiltonian.cpp:88-112)
  HostIndex h;
  h.n_qubits = n_qubits;
  h.n_words = n_words;
  std::unordered_map<WordsN, uint32_t, WordsNHash> xy_lookup;
  std::vector<std::vector<uint32_t>> members;
  for (size_t i = 0; i < keys.size(); ++i) {
    if (std::abs(mcoef[i]) < 1e-12) continue;  // kDropThreshold (hamiltonian.cpp:14, 93)
    WordsN m{};
    for (int w = 0; w < n_words; ++w) m[w] = keys[i][w] | keys[i][kMaxWords + w];
    auto [it, fresh] = xy_lookup.emplace(m, static_cast<uint32_t>(members.size()));
    if (fresh) {
      members.emplace_back();
      for (int w = 0; w < n_words; ++w) h.xy.push_back(m[w]);
    }
    members[it->second].push_back(static_cast<uint32_t>(i));
  }
  h.offsets.assign(members.size() + 1, 0);
  for (size_t g = 0; g < members.size(); ++g) {
    h.offsets[g] = h.coeff.size();
    for (uint32_t i : members[g]) {
      h.coeff.push_back(mcoef[i]);
      int yc = 0;
      for (int w = 0; w < n_words; ++w) {
        const uint64_t x = keys[i][w], y = keys[i][kMaxWords + w], z = keys[i][2 * kMaxWords + w];
        h.x.push_back(x);
        h.y.push_back(y);
        h.z.push_back(z);
        h.yz.push_back(y | z);
        yc += std::popcount(y);
      }
      h.y_weight.push_back(static_cast<uint8_t>(yc));
    }
  }
  h.offsets[members.size()] = h.coeff.size();
  const auto d = xy_lookup.find(WordsN{});
  h.diag = d == xy_lookup.end() ? -1 : static_cast<int64_t>(d->second);
  return h;
}

const uint64_t* qubit_codes() {
  static const std::array<uint64_t, 256> codes = [] {
    std::array<uint64_t, 256> c{};
    uint64_t s = 0x51A7E5B200ull;
    for (auto& v : c) v = splitmix64(s);
    return c;
  }();
  return codes.data();
}

uint32_t xy_position_key(const uint64_t* words, int n_words) {
  uint32_t key = 0xFFFFFFFFu;
  int k = 0;
  for (int w = 0; w < n_words && k < 4; ++w) {
    uint64_t v = words[w];
    while (v && k < 4) {
      const uint32_t p = static_cast<uint32_t>(w * 64 + std::countr_zero(v));
      key = (key & ~(0xFFu << (8 * k))) | (p << (8 * k));
      ++k;
      v &= v - 1;
    }
  }
  return key;
}

uint64_t linear_hash(const uint64_t* words, int n_words) {
  const uint64_t* r = qubit_codes();
  uint64_t h = 0;
  for (int w = 0; w < n_words; ++w) {
    uint64_t v = words[w];
    while (v) {
      const int b = std::countr_zero(v);
      h ^= r[w * 64 + b];
      v &= v - 1;
    }
  }
  return h;
}

std::vector<uint64_t> binomial_table() {
  constexpr uint64_t kSat = ~uint64_t{0};
  std::vector<uint64_t> c(static_cast<size_t>(257) * kBinomKHost, 0);
  for (int n = 0; n <= 256; ++n) {
    c[static_cast<size_t>(n) * kBinomKHost] = 1;
    for (int k = 1; k < kBinomKHost && n > 0; ++k) {
      const uint64_t a = c[static_cast<size_t>(n - 1) * kBinomKHost + k - 1];
      const uint64_t b = c[static_cast<size_t>(n - 1) * kBinomKHost + k];
      c[static_cast<size_t>(n) * kBinomKHost + k] = (a == kSat || b == kSat || a > kSat - b) ? kSat : a + b;
    }
  }
  return c;
}

DevicePlan plan_device(const HostIndex& h) {
  DevicePlan p;
  const int n = h.n_qubits, W = h.n_words;
  const uint32_t n_xy = h.n_xy();
  p.xy_hash.resize(n_xy);
  p.xy_weight.resize(n_xy);
  p.offsets32.resize(n_xy + 1);
  if (h.n_terms() >= 0xFFFFFFFFull) throw std::invalid_argument("HamiltonianIndex: more than 2^32-1 terms");
  for (uint32_t g = 0; g <= n_xy; ++g) p.offsets32[g] = static_cast<uint32_t>(h.offsets[g]);

  const uint32_t n_lists = static_cast<uint32_t>(n + n * (n - 1) / 2);
  std::vector<uint32_t> count(n_lists + 1, 0);
  auto for_each_list = [&](uint32_t g, auto&& fn) {
    int pos[4], k = 0;
    for (int w = 0; w < W; ++w) {
      uint64_t v = h.xy[static_cast<size_t>(g) * W + w];
      while (v && k < 4) {
        pos[k++] = w * 64 + std::countr_zero(v);
        v &= v - 1;
      }
    }
    if (p.xy_weight[g] == 2) {
      fn(static_cast<uint32_t>(pos[0]));
      fn(static_cast<uint32_t>(pos[1]));
    } else if (p.xy_weight[g] == 4) {
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b) fn(static_cast<uint32_t>(n) + pair_index(pos[a], pos[b], n));
    }
  };
  for (uint32_t g = 0; g < n_xy; ++g) {
    int wt = 0;
    for (int w = 0; w < W; ++w) wt += std::popcount(h.xy[static_cast<size_t>(g) * W + w]);
    p.xy_weight[g] = static_cast<uint8_t>(wt);
    p.xy_hash[g] = linear_hash(&h.xy[static_cast<size_t>(g) * W], W);
    if (static_cast<int64_t>(g) == h.diag) continue;
    p.gen_g.push_back(g);
    p.gen_hash.push_back(p.xy_hash[g]);
    if (wt == 2 || wt == 4)
      for_each_list(g, [&](uint32_t id) { ++count[id + 1]; });
    else if (wt % 2 == 0)
      p.res_g.push_back(g);
    // odd weights change the particle number: never inside one sector
  }
  p.lst_off.assign(n_lists + 1, 0);
  for (uint32_t i = 0; i < n_lists; ++i) p.lst_off[i + 1] = p.lst_off[i] + count[i + 1];
  p.lst_hash.resize(p.lst_off[n_lists]);
  p.lst_g.resize(p.lst_off[n_lists]);
  std::vector<uint32_t> fill(p.lst_off.begin(), p.lst_off.end() - 1);
  for (uint32_t g = 0; g < n_xy; ++g) {
    if (static_cast<int64_t>(g) == h.diag) continue;
    const int wt = p.xy_weight[g];
    if (wt != 2 && wt != 4) continue;
    for_each_list(g, [&](uint32_t id) {
      const uint32_t e = fill[id]++;
      p.lst_hash[e] = p.xy_hash[g];
      p.lst_g[e] = g;
    });
  }

  // Diagonal group: every term is a Z string (xy = 0 forces x = y = 0), so
  // its element is sum_t c_t (-1)^{|x & z_t|}. Terms with |z| <= 2 form
  // c0 + sum_p a_p s_p + sum_{p<q} J_pq s_p s_q with s_p = 1 - 2 x_p, which
  // is rewritten over the minority set S of x (occupied or empty orbitals):
  //   occupied: A + sum_{p in S} b_p + sum_{p<q in S} 4 J_pq,
  //     A = c0 + sum a + sum J, b_p = -2 a_p - 2 sum_{q!=p} J_pq
  //   holes:    A' = c0 - sum a + sum J, b'_p = 2 a_p - 2 sum_{q!=p} J_pq.
  if (h.diag >= 0) {
    p.diag_quad = true;
    long double c0 = 0, sa = 0, sj = 0;
    std::vector<long double> a(n, 0), row(n, 0);
    p.diag_K.assign(static_cast<size_t>(n) * n, 0.0);
    for (uint64_t t = h.offsets[h.diag]; t < h.offsets[h.diag + 1]; ++t) {
      if (h.y_weight[t] != 0) {  // cannot happen for xy = 0; keep exact anyway
        p.diag_other.push_back(static_cast<uint32_t>(t));
        continue;
      }
      int pos[3], k = 0;
      for (int w = 0; w < W; ++w) {
        uint64_t v = h.yz[t * W + w];
        while (v && k < 3) {
          pos[k++] = w * 64 + std::countr_zero(v);
          v &= v - 1;
        }
      }
      const long double c = h.coeff[t];
      if (k == 0) {
        c0 += c;
      } else if (k == 1) {
        a[pos[0]] += c;
        sa += c;
      } else if (k == 2) {
        p.diag_K[static_cast<size_t>(pos[0]) * n + pos[1]] += static_cast<double>(4 * c);
        p.diag_K[static_cast<size_t>(pos[1]) * n + pos[0]] += static_cast<double>(4 * c);
        row[pos[0]] += c;
        row[pos[1]] += c;
        sj += c;
      } else {
        p.diag_other.push_back(static_cast<uint32_t>(t));
      }
    }
    p.diag_A[1] = static_cast<double>(c0 + sa + sj);
    p.diag_A[0] = static_cast<double>(c0 - sa + sj);
    p.diag_b.assign(2 * static_cast<size_t>(n), 0.0);
    for (int q = 0; q < n; ++q) {
      p.diag_b[n + q] = static_cast<double>(-2 * a[q] - 2 * row[q]);
      p.diag_b[q] = static_cast<double>(2 * a[q] - 2 * row[q]);
    }
  }

  // family compression of the large groups (the 2+2(N-2)-term single
  // excitations of JW Hamiltonians: an XX and a YY family, each with one
  // optional Z dressing per term)
  p.comp_of.assign(n_xy, -1);
  p.fam_off.push_back(0);
  for (uint32_t g = 0; g < n_xy; ++g) {
    if (static_cast<int64_t>(g) == h.diag) continue;
    const uint64_t t0 = h.offsets[g], t1 = h.offsets[g + 1];
    if (t1 - t0 <= kSmallGroupHost) continue;
    struct Fam {
      std::vector<uint64_t> B;
      uint8_t q;
      long double u = 0;
      std::vector<long double> v;
    };
    // family bases: per y-weight class the bitwise majority of the terms' yz
    // masks (the undressed string, even when a Z-dressed term comes first in
    // the group, as in real molecular Hamiltonians); terms then attach to the
    // base within one bit, new bases are opened greedily if needed
    std::vector<Fam> fams;
    {
      std::vector<uint8_t> qs;
      for (uint64_t t = t0; t < t1; ++t)
        if (std::find(qs.begin(), qs.end(), h.y_weight[t] & 3) == qs.end()) qs.push_back(h.y_weight[t] & 3);
      for (uint8_t q : qs) {
        if (static_cast<int>(fams.size()) == kMaxFamilies) break;
        std::vector<uint64_t> maj(W, 0);
        uint64_t cnt = 0;
        std::vector<uint32_t> ones(static_cast<size_t>(W) * 64, 0);
        for (uint64_t t = t0; t < t1; ++t) {
          if ((h.y_weight[t] & 3) != q) continue;
          ++cnt;
          for (int w = 0; w < W; ++w)
            for (uint64_t v = h.yz[t * W + w]; v; v &= v - 1) ++ones[w * 64 + std::countr_zero(v)];
        }
        for (int b = 0; b < W * 64; ++b)
          if (2 * ones[b] > cnt) maj[b / 64] |= 1ull << (b % 64);
        fams.push_back(Fam{maj, q, 0, std::vector<long double>(n, 0)});
      }
    }
    bool ok = true;
    for (uint64_t t = t0; t < t1 && ok; ++t) {
      const uint8_t q = h.y_weight[t] & 3;
      const uint64_t* yz = &h.yz[t * W];
      int pick = -1, bitpos = -1;
      for (size_t f = 0; f < fams.size() && pick < 0; ++f) {
        if (fams[f].q != q) continue;
        int pc = 0, bp = -1;
        for (int w = 0; w < W; ++w) {
          const uint64_t d = yz[w] ^ fams[f].B[w];
          pc += std::popcount(d);
          if (d) bp = w * 64 + std::countr_zero(d);
        }
        if (pc <= 1) {
          pick = static_cast<int>(f);
          bitpos = pc ? bp : -1;
        }
      }
      if (pick < 0) {
        if (static_cast<int>(fams.size()) == kMaxFamilies) {
          ok = false;
          break;
        }
        fams.push_back(Fam{std::vector<uint64_t>(yz, yz + W), q, 0, std::vector<long double>(n, 0)});
        pick = static_cast<int>(fams.size()) - 1;
      }
      if (bitpos < 0) fams[pick].u += h.coeff[t];
      else fams[pick].v[bitpos] += h.coeff[t];
    }
    if (!ok) continue;
    p.comp_of[g] = static_cast<int32_t>(p.fam_off.size() - 1);
    for (const Fam& f : fams) {
      p.fam_B.insert(p.fam_B.end(), f.B.begin(), f.B.end());
      p.fam_q.push_back(f.q);
      p.fam_u.push_back(static_cast<double>(f.u));
      long double V = 0;
      for (int k = 0; k < n; ++k) {
        V += f.v[k];
        p.fam_v.push_back(static_cast<double>(f.v[k]));
      }
      p.fam_V.push_back(static_cast<double>(V));
    }
    p.fam_off.push_back(static_cast<uint32_t>(p.fam_q.size()));
  }

  // one-load records for the drain
  {
    const int TW = term_words(W), FW = fam_words(W);
    p.ginfo.assign(static_cast<size_t>(n_xy) * 4, 0);
    for (uint32_t g = 0; g < n_xy; ++g) {
      uint32_t* gi = &p.ginfo[static_cast<size_t>(g) * 4];
      gi[0] = static_cast<uint32_t>(h.offsets[g]);
      gi[1] = static_cast<uint32_t>(h.offsets[g + 1] - h.offsets[g]);
      gi[2] = 0xFFFFFFFFu;
      const int32_t c = p.comp_of[g];
      if (c >= 0) {
        const uint32_t f0 = p.fam_off[c], f1 = p.fam_off[c + 1];
        gi[2] = f0;
        gi[3] = f1 - f0;
        for (uint32_t f = f0; f < f1; ++f) gi[3] |= static_cast<uint32_t>(p.fam_q[f] & 3) << (8 + 2 * (f - f0));
      }
    }
    p.trec.assign(h.n_terms() * TW, 0);
    for (uint64_t t = 0; t < h.n_terms(); ++t) {
      uint64_t* r = &p.trec[t * TW];
      for (int w = 0; w < W; ++w) r[w] = h.yz[t * W + w];
      std::memcpy(&r[W], &h.coeff[t], 8);
      r[W + 1] = h.y_weight[t];
    }
    const size_t nf = p.fam_q.size();
    p.famrec.assign(nf * FW, 0);
    for (size_t f = 0; f < nf; ++f) {
      uint64_t* r = &p.famrec[f * FW];
      std::memcpy(&r[0], &p.fam_u[f], 8);
      std::memcpy(&r[1], &p.fam_V[f], 8);
      for (int w = 0; w < W; ++w) r[2 + w] = p.fam_B[f * W + w];
    }
  }

  // join-path drain records, 8 words per group (qvmc_join.cuh kGrec*):
  // A = small weight-2/4 group whose terms share one Z string (all JW double
  // excitations), B = family-compressed, C = anything else
  {
    p.grec.assign(static_cast<size_t>(n_xy) * kGrecWordsHost, 0);
    for (uint32_t g = 0; g < n_xy; ++g) {
      uint64_t* r = &p.grec[static_cast<size_t>(g) * kGrecWordsHost];
      const uint64_t t0 = h.offsets[g], t1 = h.offsets[g + 1], k = t1 - t0;
      const int32_t c = p.comp_of[g];
      const uint64_t* xy = &h.xy[static_cast<size_t>(g) * W];
      const int wt = p.xy_weight[g];
      if (c >= 0) {
        const uint32_t f0 = p.fam_off[c], f1 = p.fam_off[c + 1], nf = f1 - f0;
        uint64_t qb = 0;
        for (uint32_t f = f0; f < f1; ++f) qb |= static_cast<uint64_t>(p.fam_q[f] & 3) << (2 * (f - f0));
        // compact form: every family base B_f = (shared Z string) | (Y positions among the flip positions)
        bool compact = wt == 2 && 2 + W + 2 * static_cast<int>(nf) <= kGrecWordsHost;
        int xpos[2], np = 0;
        for (int w = 0; w < W && compact; ++w)
          for (uint64_t v = xy[w]; v && np < 2; v &= v - 1) xpos[np++] = w * 64 + std::countr_zero(v);
        uint64_t ypats = 0;
        for (uint32_t f = f0; f < f1 && compact; ++f) {
          const uint64_t* B = &p.fam_B[static_cast<size_t>(f) * W];
          for (int w = 0; w < W; ++w)
            if ((B[w] & ~xy[w]) != (p.fam_B[static_cast<size_t>(f0) * W + w] & ~xy[w])) compact = false;
          uint64_t yp = 0;
          for (int i = 0; i < np; ++i)
            if ((B[xpos[i] >> 6] >> (xpos[i] & 63)) & 1) yp |= 1ull << i;
          ypats |= yp << (4 * (f - f0));
        }
        if (compact) {
          const uint32_t nfp = nf == 1 ? 1 : nf == 2 ? 2 : 4;
          while (p.famvi.size() % 4) p.famvi.push_back(0.0);  // 32-byte aligned blocks
          r[0] = 1 | static_cast<uint64_t>(nf) << 8 | qb << 16 | ypats << 24;
          r[1] = p.famvi.size();
          for (int w = 0; w < W; ++w) r[2 + w] = p.fam_B[static_cast<size_t>(f0) * W + w] & ~xy[w];
          for (uint32_t f = f0; f < f1; ++f) {
            std::memcpy(&r[2 + W + 2 * (f - f0)], &p.fam_u[f], 8);
            std::memcpy(&r[3 + W + 2 * (f - f0)], &p.fam_V[f], 8);
          }
          for (int k = 0; k < n; ++k)
            for (uint32_t j = 0; j < nfp; ++j)
              p.famvi.push_back(j < nf ? p.fam_v[static_cast<size_t>(f0 + j) * n + k] : 0.0);
        } else {
          r[0] = 3 | static_cast<uint64_t>(nf) << 8 | qb << 16;
          r[1] = f0;
        }
        continue;
      }
      bool a_ok = static_cast<int64_t>(g) != h.diag && (wt == 2 || wt == 4) && k >= 1 &&
                  k <= static_cast<uint64_t>(kGrecWordsHost - 1 - W);
      int xpos[4], np = 0;
      for (int w = 0; w < W && a_ok; ++w)
        for (uint64_t v = xy[w]; v; v &= v - 1) xpos[np++] = w * 64 + std::countr_zero(v);
      uint64_t meta = static_cast<uint64_t>(k) << 2;
      for (uint64_t t = t0; t < t1 && a_ok; ++t) {
        const uint64_t* yz = &h.yz[t * W];
        for (int w = 0; w < W; ++w)
          if ((yz[w] & ~xy[w]) != (h.yz[t0 * W + w] & ~xy[w])) a_ok = false;  // Z strings differ
        uint64_t ypat = 0;
        for (int i = 0; i < np; ++i)
          if ((yz[xpos[i] >> 6] >> (xpos[i] & 63)) & 1) ypat |= 1ull << i;
        meta |= (ypat | static_cast<uint64_t>(h.y_weight[t] & 3) << 4) << (8 + 6 * (t - t0));
      }
      if (a_ok) {
        r[0] = meta;  // kind A = 0
        for (int w = 0; w < W; ++w) r[1 + w] = h.yz[t0 * W + w] & ~xy[w];
        for (uint64_t t = t0; t < t1; ++t) std::memcpy(&r[1 + W + (t - t0)], &h.coeff[t], 8);
      } else {
        if (k >= (1ull << 32)) throw std::invalid_argument("HamiltonianIndex: group with 2^32 or more terms");
        r[0] = 2;
        r[1] = t0 | k << 32;
      }
    }
  }

  // existence bitmaps of the weight-2/4 masks over orbital pairs (join-path
  // prefilter: a candidate's mask is looked up only when its bit is set)
  if (n <= 128) {
    const uint64_t P = static_cast<uint64_t>(n) * (n - 1) / 2;
    p.pbits_P = static_cast<uint32_t>(P);
    p.pbits.assign((P + P * P + 31) / 32, 0);
    auto pid = [](int a, int b) { return static_cast<uint64_t>(b) * (b - 1) / 2 + a; };  // a < b
    auto set = [&](uint64_t i) { p.pbits[i >> 5] |= 1u << (i & 31); };
    for (uint32_t g = 0; g < n_xy; ++g) {
      const int wt = p.xy_weight[g];
      if (static_cast<int64_t>(g) == h.diag || (wt != 2 && wt != 4)) continue;
      int q[4], k = 0;
      for (int w = 0; w < W; ++w)
        for (uint64_t v = h.xy[static_cast<size_t>(g) * W + w]; v && k < 4; v &= v - 1) q[k++] = w * 64 + std::countr_zero(v);
      if (wt == 2) {
        set(pid(q[0], q[1]));
        continue;
      }
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b) {
          int o[2], m = 0;
          for (int c = 0; c < 4; ++c)
            if (c != a && c != b) o[m++] = q[c];
          set(P + pid(q[a], q[b]) * P + pid(o[0], o[1]));
        }
    }
  }

  // flip-mask table for the join path: weight-2/4 masks keyed EXACTLY by
  // their sorted orbital positions packed into 32 bits (0xFF pads weight 2),
  // so a lookup needs no mask compare; buckets of 4 x (key32 << 32 | group),
  // chained to the next bucket when full
  {
    uint64_t nb = 64;  // about one entry per 4-slot bucket: 32 B per probe, chains ~1% of buckets
    while (nb * 2 < n_xy) nb <<= 1;
    p.xy_tab.assign(nb * 4, ~uint64_t{0});
    p.xy_tab_mask = nb - 1;
    for (uint32_t g = 0; g < n_xy; ++g) {
      const int wt = p.xy_weight[g];
      if (static_cast<int64_t>(g) == h.diag || (wt != 2 && wt != 4)) continue;
      const uint32_t key = xy_position_key(&h.xy[static_cast<size_t>(g) * W], W);
      const uint64_t entry = static_cast<uint64_t>(key) << 32 | g;
      for (uint64_t b = xy_bucket_host(key, static_cast<uint32_t>(p.xy_tab_mask));; b = (b + 1) & p.xy_tab_mask) {
        int k = 0;
        while (k < 4 && p.xy_tab[b * 4 + k] != ~uint64_t{0}) ++k;
        if (k < 4) {
          p.xy_tab[b * 4 + k] = entry;
          break;
        }
      }
    }
  }

  // byte tables of the linear hash: T[k][v] = XOR of codes of the bits of byte v at byte k
  const uint64_t* r = qubit_codes();
  p.hash_bytes.assign(static_cast<size_t>(W) * 8 * 256, 0);
  for (int k = 0; k < W * 8; ++k)
    for (int v = 0; v < 256; ++v) {
      uint64_t x = 0;
      for (int b = 0; b < 8; ++b)
        if ((v >> b) & 1) x ^= r[k * 8 + b];
      p.hash_bytes[static_cast<size_t>(k) * 256 + v] = x;
    }
  return p;
}

}  // namespace qvmc_b200
