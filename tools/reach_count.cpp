// distinct level-j states reachable from each 1/G shard of C4 (analysis only)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <set>
#include <string>
#include <cstring>
#include <algorithm>
struct K { uint32_t T, tpb, rpt, shm, A, M; };
int main(int argc, char** argv) {
  // C4 kernels passed as 72 numbers on stdin
  std::vector<K> ks(12);
  for (auto& k : ks) if (scanf("%u %u %u %u %u %u", &k.T, &k.tpb, &k.rpt, &k.shm, &k.A, &k.M) != 6) return 1;
  const int n = 12, S = 16; const uint64_t cap[4] = {32768, 49152, 48, 8};
  const int P = 7; int G = argc > 1 ? atoi(argv[1]) : 8;
  uint64_t np = 1; for (int j = 0; j < P; j++) np *= (n - j);
  std::vector<std::set<std::string>> perlev(G * (P + 1));
  std::vector<int> order(P);
  for (uint64_t p = 0; p < np; p++) {
    // unrank prefix p (lexicographic over prefixes of length P)
    uint64_t r = p; std::vector<int> L; for (int i = 0; i < n; i++) L.push_back(i);
    uint64_t f = 1; for (int j = 1; j < P; j++) f *= (n - j);
    for (int j = 0; j < P; j++) { uint64_t d = r / f; r %= f; order[j] = L[d]; L.erase(L.begin() + d); if (j + 1 < P) f /= (n - j - 1); }
    int g = (int)(p * G / np);
    std::vector<uint64_t> fr(S * 4); for (int s = 0; s < S; s++) for (int q = 0; q < 4; q++) fr[s*4+q] = cap[q];
    uint32_t cur = 0; uint64_t I = 0, M = 0; uint32_t mask = 0;
    for (int j = 0; j < P; j++) {
      const K& k = ks[order[j]]; uint64_t d[4] = {(uint64_t)k.rpt * k.tpb, k.shm, (k.tpb + 31) / 32, 1};
      for (uint32_t b = 0; b < k.T; b++) {
        int found = -1;
        for (int st = 0; st < S; st++) { int s = (cur + st) % S; bool ok = true; for (int q = 0; q < 4; q++) ok &= d[q] <= fr[s*4+q]; if (ok) { found = s; break; } }
        if (found < 0) { for (int s = 0; s < S; s++) for (int q = 0; q < 4; q++) fr[s*4+q] = cap[q]; cur = 0; I = M = 0; found = 0; }
        for (int q = 0; q < 4; q++) fr[found*4+q] -= d[q];
        I += k.A; M += k.M; cur = (found + 1) % S;
      }
      mask |= 1u << order[j];
      std::string key((char*)fr.data(), fr.size() * 8); key.append((char*)&cur, 4); key.append((char*)&I, 8); key.append((char*)&M, 8); key.append((char*)&mask, 4);
      perlev[g * (P + 1) + j + 1].insert(key);
    }
  }
  for (int j = 1; j <= P; j++) { printf("level %d:", j); std::set<std::string> all; for (int g = 0; g < G; g++) { printf(" %zu", perlev[g*(P+1)+j].size()); for (auto& x : perlev[g*(P+1)+j]) all.insert(x);} printf(" | all %zu\n", all.size()); }
}
