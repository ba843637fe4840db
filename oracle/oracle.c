/* oracle.c — CPU restatement of the reference's traversal algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  Used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py as the checker and the CPU
 * baseline; never linked into or called by the product library (libgg.so).
 *
 * Every function follows the reference package `schedge`
 * (/root/reference/pkg/src/schedge/, cited file:line) with the same
 * semantics; pinned against fixtures produced by the reference itself
 * (tests/golden/, made by oracle/make_golden.py).
 *
 * Build: make -C oracle   (liboracle.so, gcc -O3 -fopenmp)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

#define UNREACHED UINT64_MAX /* priority.py:14 */

int or_num_threads(void) { return omp_get_max_threads(); }

/* graphio._build_csr (graphio.py:95-102): stable counting sort of keys->vals. */
void or_build_csr(int64_t V, int64_t E, const int32_t* keys, const int32_t* vals,
                  const uint32_t* w, int64_t* off, int32_t* nbr, uint32_t* wout) {
  memset(off, 0, (V + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < E; ++i) off[keys[i] + 1]++;
  for (int64_t v = 0; v < V; ++v) off[v + 1] += off[v];
  int64_t* cur = (int64_t*)malloc((V + 1) * sizeof(int64_t));
  memcpy(cur, off, (V + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < E; ++i) {
    int64_t p = cur[keys[i]]++;
    nbr[p] = vals[i];
    if (w && wout) wout[p] = w[i];
  }
  free(cur);
}

/* algos.pagerank (algos.py:163-208) with the default EDGE_ONLY schedule:
 * acc[dst] += contrib[src] in COO order, f64 throughout.  Returns iterations. */
int64_t or_pagerank(int64_t V, int64_t E, const int32_t* src, const int32_t* dst,
                    int64_t max_iters, double tol, double damping, double* rank) {
  int64_t* deg = (int64_t*)calloc(V, sizeof(int64_t));
  double* acc = (double*)calloc(V, sizeof(double));
  double* contrib = (double*)calloc(V, sizeof(double));
  for (int64_t i = 0; i < E; ++i) deg[src[i]]++;
  for (int64_t v = 0; v < V; ++v) rank[v] = 1.0 / (double)V;
  int64_t iters = 0;
  double l1 = INFINITY;
  while (!(iters >= max_iters || l1 < tol)) {
    double dm = 0.0;
    for (int64_t v = 0; v < V; ++v)
      if (!deg[v]) dm += rank[v];
    for (int64_t v = 0; v < V; ++v) contrib[v] = deg[v] ? rank[v] / (double)deg[v] : 0.0;
    for (int64_t i = 0; i < E; ++i) acc[dst[i]] += contrib[src[i]];
    double base = (1.0 - damping) / (double)V + damping * dm / (double)V;
    l1 = 0.0;
    for (int64_t v = 0; v < V; ++v) {
      double nv = base + damping * acc[v];
      l1 += fabs(nv - rank[v]);
      rank[v] = nv;
      acc[v] = 0.0;
    }
    iters++;
  }
  free(deg);
  free(acc);
  free(contrib);
  return iters;
}

/* Same iteration, parallel over destinations (pull over CSR-in, OpenMP):
 * the multi-core CPU baseline.  Summation order per vertex = CSR-in order. */
int64_t or_pagerank_par(int64_t V, const int64_t* in_off, const int32_t* in_nbr,
                        const int64_t* out_off, int64_t max_iters, double tol, double damping,
                        double* rank) {
  double* contrib = (double*)malloc(V * sizeof(double));
  double* next = (double*)malloc(V * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) rank[v] = 1.0 / (double)V;
  int64_t iters = 0;
  double l1 = INFINITY;
  while (!(iters >= max_iters || l1 < tol)) {
    double dm = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : dm)
    for (int64_t v = 0; v < V; ++v) {
      int64_t d = out_off[v + 1] - out_off[v];
      contrib[v] = d ? rank[v] / (double)d : 0.0;
      if (!d) dm += rank[v];
    }
    double base = (1.0 - damping) / (double)V + damping * dm / (double)V;
    l1 = 0.0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : l1)
    for (int64_t v = 0; v < V; ++v) {
      double s = 0.0;
      for (int64_t e = in_off[v]; e < in_off[v + 1]; ++e) s += contrib[in_nbr[e]];
      double nv = base + damping * s;
      l1 += fabs(nv - rank[v]);
      next[v] = nv;
    }
    memcpy(rank, next, V * sizeof(double));
    iters++;
  }
  free(contrib);
  free(next);
  return iters;
}

/* BFS hop levels from `source` (reference semantics: bfs + bfs_levels,
 * algos.py:101-156; levels are schedule-independent).  -1 unreached. */
void or_bfs_levels(int64_t V, const int64_t* off, const int32_t* nbr, int64_t source,
                   int32_t* level) {
  for (int64_t v = 0; v < V; ++v) level[v] = -1;
  int32_t* q = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  int64_t head = 0, tail = 0;
  level[source] = 0;
  q[tail++] = (int32_t)source;
  while (head < tail) {
    int32_t u = q[head++];
    for (int64_t e = off[u]; e < off[u + 1]; ++e) {
      int32_t v = nbr[e];
      if (level[v] == -1) {
        level[v] = level[u] + 1;
        q[tail++] = v;
      }
    }
  }
  free(q);
}

/* Parallel level-synchronous BFS (OpenMP, top-down): multi-core baseline. */
void or_bfs_levels_par(int64_t V, const int64_t* off, const int32_t* nbr, int64_t source,
                       int32_t* level) {
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) level[v] = -1;
  int32_t* cur = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  int32_t* nxt = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  int64_t ncur = 1, d = 0;
  cur[0] = (int32_t)source;
  level[source] = 0;
  while (ncur) {
    int64_t nn = 0;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < ncur; ++i) {
      int32_t u = cur[i];
      for (int64_t e = off[u]; e < off[u + 1]; ++e) {
        int32_t v = nbr[e];
        if (level[v] == -1 && __sync_bool_compare_and_swap(&level[v], -1, (int32_t)(d + 1))) {
          int64_t p = __sync_fetch_and_add(&nn, 1);
          nxt[p] = v;
        }
      }
    }
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
    ncur = nn;
    d++;
  }
  free(cur);
  free(nxt);
}

/* Delta-stepping SSSP with the reference's two-bucket queue
 * (priority.py:17-118, algos.py:215-247): current bucket [i*delta,(i+1)*delta),
 * far bucket with lazy re-bucketing, stale entries filtered on advance.
 * dist: UINT64_MAX for unreached.  Returns the number of body rounds
 * (relax rounds + advance rounds, as counted by fused_loop). */
int64_t or_sssp_delta(int64_t V, const int64_t* off, const int32_t* nbr, const uint32_t* w,
                      int64_t source, int64_t delta, uint64_t* dist) {
  for (int64_t v = 0; v < V; ++v) dist[v] = UNREACHED;
  int64_t cap = V > 0 ? V : 1;
  int32_t* cur = (int32_t*)malloc(cap * sizeof(int32_t));
  int32_t* take = (int32_t*)malloc(cap * sizeof(int32_t));
  int32_t* far = (int32_t*)malloc(cap * sizeof(int32_t));
  int32_t* far2 = (int32_t*)malloc(cap * sizeof(int32_t));
  uint8_t* cmark = (uint8_t*)calloc(cap, 1);
  uint8_t* fmark = (uint8_t*)calloc(cap, 1);
  int64_t ncur = 0, nfar = 0, rounds = 0;
  uint64_t index;
  dist[source] = 0; /* seed (priority.py:35-39) */
  index = 0 / (uint64_t)delta;
  cur[ncur++] = (int32_t)source;
  cmark[source] = 1;
  while (!(ncur == 0 && nfar == 0)) {
    rounds++;
    if (ncur == 0) { /* advance (priority.py:85-115) */
      for (int64_t i = 0; i < nfar; ++i) fmark[far[i]] = 0;
      uint64_t best = UINT64_MAX;
      int64_t n2 = 0;
      for (int64_t i = 0; i < nfar; ++i) {
        uint64_t b = dist[far[i]] / (uint64_t)delta;
        if (b <= index) continue;
        far2[n2++] = far[i];
        if (b < best) best = b;
      }
      nfar = 0;
      if (best == UINT64_MAX) continue;
      index = best;
      for (int64_t i = 0; i < n2; ++i) {
        int32_t v = far2[i];
        uint64_t b = dist[v] / (uint64_t)delta;
        if (b == best) {
          if (!cmark[v]) { cmark[v] = 1; cur[ncur++] = v; }
        } else if (!fmark[v]) {
          fmark[v] = 1;
          far[nfar++] = v;
        }
      }
      continue;
    }
    /* take_current + relax (algos.py:240-243) */
    int64_t nt = ncur;
    memcpy(take, cur, nt * sizeof(int32_t));
    for (int64_t i = 0; i < nt; ++i) cmark[take[i]] = 0;
    ncur = 0;
    for (int64_t i = 0; i < nt; ++i) {
      int32_t u = take[i];
      for (int64_t e = off[u]; e < off[u + 1]; ++e) {
        int32_t v = nbr[e];
        uint64_t cand = dist[u] + (uint64_t)w[e];
        if (cand >= dist[v]) continue;
        dist[v] = cand;
        if (cand / (uint64_t)delta == index) {
          if (!cmark[v]) { cmark[v] = 1; cur[ncur++] = v; }
        } else if (!fmark[v]) {
          fmark[v] = 1;
          far[nfar++] = v;
        }
      }
    }
  }
  free(cur); free(take); free(far); free(far2); free(cmark); free(fmark);
  return rounds;
}

/* cc_soman (algos.py:267-307): hook every COO arc (label[hi] = min), full
 * pointer jumping, repeat until no hook changed; canonical min-id labels.
 * Returns the number of rounds. */
int64_t or_cc(int64_t V, int64_t E, const int32_t* src, const int32_t* dst, int32_t* out) {
  int32_t* label = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  for (int64_t v = 0; v < V; ++v) label[v] = (int32_t)v;
  int changed = 1;
  int64_t rounds = 0;
  while (changed) {
    changed = 0;
    for (int64_t i = 0; i < E; ++i) {
      int32_t la = label[src[i]], lb = label[dst[i]];
      if (la == lb) continue;
      int32_t lo = la < lb ? la : lb, hi = la < lb ? lb : la;
      if (lo < label[hi]) { label[hi] = lo; changed = 1; }
    }
    int moved = 1; /* _pointer_jump (algos.py:254-264) */
    while (moved) {
      moved = 0;
      for (int64_t v = 0; v < V; ++v) {
        int32_t l = label[v], ll = label[l];
        if (ll != l) { label[v] = ll; moved = 1; }
      }
    }
    rounds++;
  }
  /* canonicalise: first (minimum) member of each label class */
  int32_t* first = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  for (int64_t v = 0; v < V; ++v) first[v] = -1;
  for (int64_t v = 0; v < V; ++v)
    if (first[label[v]] == -1) first[label[v]] = (int32_t)v;
  for (int64_t v = 0; v < V; ++v) out[v] = first[label[v]];
  free(first);
  free(label);
  return rounds;
}

/* bc (algos.py:314-395): per source, forward level rounds with path counts
 * (f64), backward rounds over levels len-2..0 accumulating
 * delta[u] += sigma[u]/sigma[v]*(1+delta[v]) for depth[v] == depth[u]+1;
 * scores summed over sources excluding the source itself, then halved. */
void or_bc(int64_t V, const int64_t* off, const int32_t* nbr, const int64_t* sources,
           int64_t nsrc, double* score) {
  int32_t* depth = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  double* sigma = (double*)malloc((V > 0 ? V : 1) * sizeof(double));
  double* delta = (double*)malloc((V > 0 ? V : 1) * sizeof(double));
  int32_t* order = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  int64_t* lvl_start = (int64_t*)malloc((V + 2) * sizeof(int64_t));
  for (int64_t v = 0; v < V; ++v) score[v] = 0.0;
  for (int64_t si = 0; si < nsrc; ++si) {
    int64_t s = sources[si];
    for (int64_t v = 0; v < V; ++v) { depth[v] = -1; sigma[v] = 0.0; delta[v] = 0.0; }
    depth[s] = 0;
    sigma[s] = 1.0;
    int64_t n = 0, nl = 0;
    order[n++] = (int32_t)s;
    lvl_start[nl++] = 0;
    int64_t lo = 0;
    while (lo < n) { /* one round per level */
      int64_t hi = n;
      int32_t level = depth[order[lo]];
      for (int64_t i = lo; i < hi; ++i) {
        int32_t u = order[i];
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
          int32_t v = nbr[e];
          if (depth[v] == -1) { depth[v] = level + 1; order[n++] = v; }
          if (depth[v] == level + 1) sigma[v] += sigma[u];
        }
      }
      lo = hi;
      lvl_start[nl++] = n;
    }
    /* backward: levels nl-3 .. 0 as sources of the wave (rounds[len-2..0]) */
    int64_t nrounds = nl - 1; /* number of non-empty level frontiers */
    for (int64_t r = nrounds - 2; r >= 0; --r) {
      for (int64_t i = lvl_start[r]; i < lvl_start[r + 1]; ++i) {
        int32_t u = order[i];
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
          int32_t v = nbr[e];
          if (depth[v] == depth[u] + 1) delta[u] += sigma[u] / sigma[v] * (1.0 + delta[v]);
        }
      }
    }
    for (int64_t v = 0; v < V; ++v)
      if (v != s) score[v] += delta[v];
  }
  for (int64_t v = 0; v < V; ++v) score[v] /= 2.0;
  free(depth); free(sigma); free(delta); free(order); free(lvl_start);
}

/* block_edges Alg. 1 (blocking.py:78-113): stable partition by dst / n.
 * perm[k] = original edge index at blocked position k; seg_end = inclusive
 * segment ends (blocking.py:24-30). */
void or_block_edges(int64_t V, int64_t E, const int32_t* dst, int64_t n, int64_t* perm,
                    int64_t* seg_end) {
  int64_t S = (V + n - 1) / n;
  int64_t* cursor = (int64_t*)calloc(S + 1, sizeof(int64_t));
  for (int64_t i = 0; i < E; ++i) cursor[dst[i] / n]++;
  int64_t total = 0;
  for (int64_t s = 0; s < S; ++s) { int64_t c = cursor[s]; cursor[s] = total; total += c; }
  for (int64_t i = 0; i < E; ++i) perm[cursor[dst[i] / n]++] = i;
  for (int64_t s = 0; s < S; ++s) seg_end[s] = cursor[s];
  free(cursor);
}

/* Host replica of the device RMAT generator (csrc/graph.cu k_rmat), OpenMP:
 * lets the CPU baselines build their bounded samples without the GPU. */
static inline uint64_t or_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void or_rmat(int scale, int64_t E, double a, double b, double c, uint64_t seed, int32_t* src,
             int32_t* dst) {
  const double s32 = 4294967296.0;
  double t1 = a * s32, t2 = (a + b) * s32, t3 = (a + b + c) * s32;
  uint32_t ta = t1 >= s32 ? 0xffffffffu : (uint32_t)t1;
  uint32_t tab = t2 >= s32 ? 0xffffffffu : (uint32_t)t2;
  uint32_t tabc = t3 >= s32 ? 0xffffffffu : (uint32_t)t3;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < E; ++i) {
    uint32_t s = 0, d = 0;
    uint64_t h = 0;
    for (int l = 0; l < scale; ++l) {
      if ((l & 1) == 0) h = or_mix64(seed ^ or_mix64((uint64_t)i * 64 + l));
      uint32_t r = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
      uint32_t bs = r >= tab, bd = (r >= ta && r < tab) || r >= tabc;
      s = (s << 1) | bs;
      d = (d << 1) | bd;
    }
    src[i] = (int32_t)s;
    dst[i] = (int32_t)d;
  }
}

/* ------------------------------------------------------------------------
 * Full-scale parity helpers (OpenMP).  Same results as the serial
 * restatements above wherever the result is order-independent: CSR
 * neighbour order within a vertex is unspecified (atomic scatter), BFS
 * levels / CC canonical labels / SSSP distances are unique, and the BC and
 * PageRank sums differ only in summation order (checked against the serial
 * versions in tests/test_oracle_golden.py).  Used by bench.py's parity and
 * cpu_baseline legs at the BASELINE sizes, where the serial ones take minutes.
 * ------------------------------------------------------------------------ */

/* offsets of a CSR keyed by keys[] (graphio.py:95-102, counts only) */
void or_offsets_par(int64_t V, int64_t E, const int32_t* keys, int64_t* off) {
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v <= V; ++v) off[v] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < E; ++i) __atomic_fetch_add(&off[keys[i] + 1], 1, __ATOMIC_RELAXED);
  for (int64_t v = 0; v < V; ++v) off[v + 1] += off[v];
}

/* CSR keys -> vals with neighbour order within a key unspecified. */
void or_build_csr_par(int64_t V, int64_t E, const int32_t* keys, const int32_t* vals,
                      const uint32_t* w, int64_t* off, int32_t* nbr, uint32_t* wout) {
  or_offsets_par(V, E, keys, off);
  int64_t* cur = (int64_t*)malloc((V + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v <= V; ++v) cur[v] = off[v];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < E; ++i) {
    int64_t p = __atomic_fetch_add(&cur[keys[i]], 1, __ATOMIC_RELAXED);
    nbr[p] = vals[i];
    if (w && wout) wout[p] = w[i];
  }
  free(cur);
}

/* Direction-optimising BFS levels (top-down over a byte frontier, bottom-up
 * over the in-adjacency when the frontier is large).  Levels are unique, so
 * this equals or_bfs_levels for any switch rule.  Returns the level count. */
int64_t or_bfs_levels_do(int64_t V, const int64_t* off, const int32_t* nbr,
                         const int64_t* in_off, const int32_t* in_nbr, int64_t source,
                         int32_t* level) {
  uint8_t* cur = (uint8_t*)calloc(V > 0 ? V : 1, 1);
  uint8_t* nxt = (uint8_t*)calloc(V > 0 ? V : 1, 1);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) level[v] = -1;
  level[source] = 0;
  cur[source] = 1;
  int64_t nf = 1, d = 0;
  while (nf) {
    int64_t cnt = 0;
    if (nf * 20 > V) { /* bottom-up */
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : cnt)
      for (int64_t v = 0; v < V; ++v) {
        if (level[v] != -1) continue;
        for (int64_t e = in_off[v]; e < in_off[v + 1]; ++e)
          if (cur[in_nbr[e]]) { level[v] = (int32_t)(d + 1); nxt[v] = 1; cnt++; break; }
      }
    } else { /* top-down */
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : cnt)
      for (int64_t u = 0; u < V; ++u) {
        if (!cur[u]) continue;
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
          int32_t v = nbr[e];
          if (level[v] == -1 && __sync_bool_compare_and_swap(&level[v], -1, (int32_t)(d + 1))) {
            nxt[v] = 1;
            cnt++;
          }
        }
      }
    }
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < V; ++v) cur[v] = 0;
    uint8_t* t = cur; cur = nxt; nxt = t;
    nf = cnt;
    d++;
  }
  free(cur);
  free(nxt);
  return d;
}

/* BFS parent-tree legality (test_algos.py:55-62): the
 * source is its own parent, exactly the reached vertices have parents, each
 * parent sits one level above its child and the arc parent->child exists
 * (looked up in the child's in-adjacency).  Returns the number of
 * violating vertices (0 = legal). */
int64_t or_bfs_check_tree(int64_t V, const int64_t* in_off, const int32_t* in_nbr,
                          int64_t source, const int32_t* parent, const int32_t* level) {
  int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : bad)
  for (int64_t v = 0; v < V; ++v) {
    int32_t p = parent[v];
    if (v == source) { bad += (p != source); continue; }
    if (level[v] == -1) { bad += (p != -1); continue; }
    if (p < 0 || p >= V || level[p] != level[v] - 1) { bad++; continue; }
    int found = 0;
    for (int64_t e = in_off[v]; e < in_off[v + 1] && !found; ++e) found = (in_nbr[e] == p);
    bad += !found;
  }
  return bad;
}

/* cc_soman result (algos.py:267-307) by parallel hooking (atomic min on the
 * higher label, as the reference's hook) + pointer jumping to a fixpoint;
 * the canonical labels (component minimum id) are unique, so they equal
 * or_cc's.  Returns the number of hooking rounds. */
int64_t or_cc_par(int64_t V, int64_t E, const int32_t* src, const int32_t* dst, int32_t* out) {
  int32_t* label = out;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) label[v] = (int32_t)v;
  int64_t rounds = 0;
  int changed = 1;
  while (changed) {
    changed = 0;
#pragma omp parallel for schedule(static) reduction(| : changed)
    for (int64_t i = 0; i < E; ++i) {
      int32_t la = label[src[i]], lb = label[dst[i]];
      if (la == lb) continue;
      int32_t lo = la < lb ? la : lb, hi = la < lb ? lb : la;
      int32_t cur = __atomic_load_n(&label[hi], __ATOMIC_RELAXED);
      while (lo < cur) {
        if (__atomic_compare_exchange_n(&label[hi], &cur, lo, 0, __ATOMIC_RELAXED,
                                        __ATOMIC_RELAXED)) { changed = 1; break; }
      }
    }
    int moved = 1;
    while (moved) {
      moved = 0;
#pragma omp parallel for schedule(static) reduction(| : moved)
      for (int64_t v = 0; v < V; ++v) {
        int32_t l = label[v], ll = label[l];
        if (ll != l) { label[v] = ll; moved = 1; }
      }
    }
    rounds++;
  }
  return rounds; /* every label is now its component's minimum id (a root) */
}

/* bc (algos.py:314-395) level-synchronously in pull form: sigma[v] = sum of
 * sigma over in-neighbours one level up, then
 * delta[u] = sum over out-neighbours v one level down of sigma[u]/sigma[v]*(1+delta[v])
 * — the same terms as the reference's push rounds (duplicates counted per
 * arc), summed in a different order. */
void or_bc_par(int64_t V, const int64_t* off, const int32_t* nbr, const int64_t* in_off,
               const int32_t* in_nbr, const int64_t* sources, int64_t nsrc, double* score) {
  int32_t* depth = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
  double* sigma = (double*)malloc((V > 0 ? V : 1) * sizeof(double));
  double* delta = (double*)malloc((V > 0 ? V : 1) * sizeof(double));
  int32_t* order = (int32_t*)malloc((V > 0 ? V : 1) * sizeof(int32_t));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) score[v] = 0.0;
  for (int64_t si = 0; si < nsrc; ++si) {
    int64_t s = sources[si];
    int64_t nl = or_bfs_levels_do(V, off, nbr, in_off, in_nbr, s, depth);
    int64_t* start = (int64_t*)calloc(nl + 2, sizeof(int64_t));
    for (int64_t v = 0; v < V; ++v)
      if (depth[v] >= 0) start[depth[v] + 1]++;
    for (int64_t l = 0; l < nl; ++l) start[l + 1] += start[l];
    int64_t* cur = (int64_t*)malloc((nl + 1) * sizeof(int64_t));
    memcpy(cur, start, (nl + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < V; ++v)
      if (depth[v] >= 0) order[cur[depth[v]]++] = (int32_t)v;
    free(cur);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < V; ++v) { sigma[v] = 0.0; delta[v] = 0.0; }
    sigma[s] = 1.0;
    for (int64_t l = 1; l < nl; ++l) {
#pragma omp parallel for schedule(dynamic, 256)
      for (int64_t i = start[l]; i < start[l + 1]; ++i) {
        int32_t v = order[i];
        double sg = 0.0;
        for (int64_t e = in_off[v]; e < in_off[v + 1]; ++e)
          if (depth[in_nbr[e]] == l - 1) sg += sigma[in_nbr[e]];
        sigma[v] = sg;
      }
    }
    for (int64_t l = nl - 2; l >= 0; --l) {
#pragma omp parallel for schedule(dynamic, 256)
      for (int64_t i = start[l]; i < start[l + 1]; ++i) {
        int32_t u = order[i];
        double dl = 0.0;
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
          int32_t v = nbr[e];
          if (depth[v] == l + 1) dl += sigma[u] / sigma[v] * (1.0 + delta[v]);
        }
        delta[u] = dl;
      }
    }
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < V; ++v)
      if (v != s) score[v] += delta[v];
    free(start);
  }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) score[v] /= 2.0;
  free(depth); free(sigma); free(delta); free(order);
}
