/* Graph oracle in C (test infrastructure only; never linked into the product path): BFS levels,
 * SpMV and PageRank over a CSR, restated sequentially so the GPU's paged BFS / SpMV can be checked
 * at the BASELINE scales (RMAT 26: 1.07 G edges, RMAT 27: 2.15 G edges) where numpy would need
 * tens of GB of temporaries.  No reference ancestor (SPEC.md:9 drops the graph apps); parity is
 * BFS levels bit-exact and fp32 row sums within 1e-5 relative (north_star).
 *
 *   gcc -O3 -fopenmp -fPIC -shared -o oracle/_build/libgraph_oracle.so oracle/graph_oracle.c   (build())
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Level-synchronous top-down BFS with a FIFO queue: level[v] = hops from source, -1 unreached. */
int64_t oracle_bfs(const int64_t* row_ptr, const int32_t* col, int64_t V, int64_t source, int32_t* level) {
  for (int64_t v = 0; v < V; ++v) level[v] = -1;
  int32_t* q = (int32_t*)malloc((size_t)V * sizeof(int32_t));
  if (!q) return -1;
  int64_t head = 0, tail = 0, levels = 0;
  level[source] = 0;
  q[tail++] = (int32_t)source;
  while (head < tail) {
    const int32_t u = q[head++];
    const int32_t lu = level[u];
    if (lu + 1 > levels) levels = lu + 1;
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      const int32_t w = col[e];
      if (level[w] < 0) {
        level[w] = lu + 1;
        q[tail++] = w;
      }
    }
  }
  free(q);
  return levels;
}

/* y[r] = fp32(alpha * sum_e fp64(val[e]) * fp64(x[col[e]]) + beta), sums in fp64 in edge order;
 * val == NULL: unit weights. */
void oracle_spmv(const int64_t* row_ptr, const int32_t* col, const float* val, const float* x, int64_t V,
                 float alpha, float beta, float* y) {
  /* rows are independent: host threads split them (each row's sum keeps its sequential order) */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < V; ++r) {
    double s = 0.0;
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e)
      s += (val ? (double)val[e] : 1.0) * (double)x[col[e]];
    y[r] = (float)((double)alpha * s + (double)beta);
  }
}

/* PageRank on the in-edge CSR (rowT, colT), iters power steps with the GPU driver's fp32 state
 * (bench/graph.py run_pagerank): x = fp32(r * fp32(1 / outdeg)) (0 for sinks),
 * r = fp32(fp32(d) * sum_{u in in(v)} x[u] + fp32((1 - d) / V)). */
void oracle_pagerank(const int64_t* rowT, const int32_t* colT, const int64_t* outdeg, int64_t V, int iters, double d,
                     float* r) {
  float* x = (float*)malloc((size_t)V * sizeof(float));
  if (!x) return;
  for (int64_t v = 0; v < V; ++v) r[v] = (float)(1.0 / (double)V);
  const float alpha = (float)d, base = (float)((1.0 - d) / (double)V);
  for (int it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < V; ++v) x[v] = outdeg[v] > 0 ? r[v] * (1.0f / (float)outdeg[v]) : 0.0f;
    oracle_spmv(rowT, colT, NULL, x, V, alpha, base, r);
  }
  free(x);
}
