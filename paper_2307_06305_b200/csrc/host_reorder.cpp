// Host-side bandwidth reduction for the DA-CSR path (C++, CPU only).
//
// Bit-exact with the reference's reverse Cuthill–McKee
// (/root/reference/pkg/src/dacsr/reorder.py:146-197): same graph (pattern of
// A + A^T without self-loops, reorder.py:70-97), same component discovery
// (BFS from the lowest unvisited index), same George–Liu pseudo-peripheral
// start (reorder.py:126-143), same (degree, index) tie-breaking, same
// concatenation by ascending start node and final reversal.  The reference
// runs this as a pure-Python BFS (~92 s at config C4); this is O(nnz log d).
//
// permute_symmetric (reorder.py:200-220): row r of P A P^T is old row
// perm[r] with columns relabelled through inv and re-sorted.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "dacsr_b200.h"

namespace {

struct Graph {
  int64_t n;
  const int64_t* ptr;
  const int64_t* adj;
  std::vector<int64_t> degree;
};

// Breadth-first sweep from `root` over unvisited (depth < 0) vertices;
// appends the visit order to `visit` and returns the deepest level.
int64_t sweep(const Graph& g, int64_t root, std::vector<int64_t>& depth,
              std::vector<int64_t>& visit) {
  visit.clear();
  visit.push_back(root);
  depth[root] = 0;
  int64_t deepest = 0;
  for (size_t head = 0; head < visit.size(); ++head) {
    const int64_t u = visit[head];
    const int64_t next = depth[u] + 1;
    for (int64_t k = g.ptr[u]; k < g.ptr[u + 1]; ++k) {
      const int64_t w = g.adj[k];
      if (depth[w] >= 0) continue;
      depth[w] = next;
      deepest = std::max(deepest, next);
      visit.push_back(w);
    }
  }
  return deepest;
}

bool lighter(const Graph& g, int64_t a, int64_t b) {
  return g.degree[a] != g.degree[b] ? g.degree[a] < g.degree[b] : a < b;
}

int64_t lightest(const Graph& g, const std::vector<int64_t>& nodes) {
  return *std::min_element(nodes.begin(), nodes.end(),
                           [&](int64_t a, int64_t b) { return lighter(g, a, b); });
}

void clear_depth(const std::vector<int64_t>& visit, std::vector<int64_t>& depth) {
  for (int64_t u : visit) depth[u] = -1;
}

int64_t peripheral_start(const Graph& g, const std::vector<int64_t>& component,
                         std::vector<int64_t>& depth, std::vector<int64_t>& visit) {
  int64_t best = lightest(g, component);
  int64_t ecc = sweep(g, best, depth, visit);
  std::vector<int64_t> rim;
  for (int64_t u : visit)
    if (depth[u] == ecc) rim.push_back(u);
  clear_depth(visit, depth);
  for (;;) {
    const int64_t cand = lightest(g, rim);
    const int64_t ecc_c = sweep(g, cand, depth, visit);
    if (ecc_c <= ecc) {
      clear_depth(visit, depth);
      return best;
    }
    rim.clear();
    for (int64_t u : visit)
      if (depth[u] == ecc_c) rim.push_back(u);
    clear_depth(visit, depth);
    best = cand;
    ecc = ecc_c;
  }
}

}  // namespace

extern "C" {

int dacsr_host_adjacency(int64_t n, const int64_t* rowptr, const int64_t* colids, int64_t* indptr,
                         int64_t* indices) {
  if (n < 0 || !rowptr || !indptr) return DACSR_ERR_ARG;
  // neighbour lists of A + A^T (with repeats), then sort + dedupe per vertex
  std::vector<int64_t> deg(n + 1, 0);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      const int64_t c = colids[k];
      if (c == r) continue;
      ++deg[r];
      ++deg[c];
    }
  std::vector<int64_t> start(n + 1, 0);
  for (int64_t u = 0; u < n; ++u) start[u + 1] = start[u] + deg[u];
  std::vector<int64_t> buf(start[n]);
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      const int64_t c = colids[k];
      if (c == r) continue;
      buf[fill[r]++] = c;
      buf[fill[c]++] = r;
    }
  indptr[0] = 0;
  int64_t out = 0;
  for (int64_t u = 0; u < n; ++u) {
    int64_t* b = buf.data() + start[u];
    int64_t* e = buf.data() + start[u + 1];
    std::sort(b, e);
    e = std::unique(b, e);
    if (indices) std::copy(b, e, indices + out);
    out += e - b;
    indptr[u + 1] = out;
  }
  return DACSR_OK;
}

int dacsr_host_rcm(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* perm) {
  if (n < 0 || (n > 0 && (!indptr || !perm))) return DACSR_ERR_ARG;
  if (n == 0) return DACSR_OK;
  Graph g{n, indptr, indices, std::vector<int64_t>(n)};
  for (int64_t u = 0; u < n; ++u) g.degree[u] = indptr[u + 1] - indptr[u];

  std::vector<int64_t> depth(n, -1), visit;
  visit.reserve(n);
  std::vector<char> seen(n, 0);
  std::vector<int64_t> starts;
  for (int64_t s = 0; s < n; ++s) {
    if (seen[s]) continue;
    sweep(g, s, depth, visit);
    std::vector<int64_t> component(visit);
    for (int64_t u : component) seen[u] = 1;
    clear_depth(component, depth);
    starts.push_back(peripheral_start(g, component, depth, visit));
  }
  std::sort(starts.begin(), starts.end());  // components by ascending start

  std::vector<char> placed(n, 0);
  std::vector<int64_t> order;
  order.reserve(n);
  std::vector<int64_t> fresh;
  for (int64_t s : starts) {
    size_t head = order.size();
    order.push_back(s);
    placed[s] = 1;
    for (; head < order.size(); ++head) {
      const int64_t u = order[head];
      fresh.clear();
      for (int64_t k = indptr[u]; k < indptr[u + 1]; ++k)
        if (!placed[indices[k]]) fresh.push_back(indices[k]);
      std::sort(fresh.begin(), fresh.end(), [&](int64_t a, int64_t b) { return lighter(g, a, b); });
      for (int64_t w : fresh) {
        placed[w] = 1;
        order.push_back(w);
      }
    }
  }
  for (int64_t k = 0; k < n; ++k) perm[k] = order[n - 1 - k];
  return DACSR_OK;
}

int dacsr_host_permute(int64_t n, const int64_t* rowptr, const int64_t* colids, const void* values,
                       int32_t vb, const int64_t* perm, int64_t* out_rowptr, int64_t* out_colids,
                       void* out_values) {
  if (n < 0 || !rowptr || !perm || !out_rowptr || (vb != 4 && vb != 8)) return DACSR_ERR_ARG;
  std::vector<int64_t> inv(n);
  for (int64_t k = 0; k < n; ++k) {
    if (perm[k] < 0 || perm[k] >= n) return DACSR_ERR_ARG;
    inv[perm[k]] = k;
  }
  out_rowptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t old = perm[r];
    out_rowptr[r + 1] = out_rowptr[r] + (rowptr[old + 1] - rowptr[old]);
  }
  const char* vin = static_cast<const char*>(values);
  char* vout = static_cast<char*>(out_values);
  std::vector<std::pair<int64_t, int64_t>> row;  // (new column, source entry)
  for (int64_t r = 0; r < n; ++r) {
    const int64_t old = perm[r];
    row.clear();
    for (int64_t k = rowptr[old]; k < rowptr[old + 1]; ++k) row.emplace_back(inv[colids[k]], k);
    std::sort(row.begin(), row.end());
    int64_t at = out_rowptr[r];
    for (const auto& [c, k] : row) {
      out_colids[at] = c;
      std::memcpy(vout + at * vb, vin + k * vb, vb);
      ++at;
    }
  }
  return DACSR_OK;
}

}  // extern "C"
