// Probe: phase timing of the gain kernel (chol_logdet_kernel) on a batch of
// SPD blocks, via clock64 stamps (thread 0 of block 0).
#define DSEL_PROBE 1
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>
__device__ long long g_stamps[128];
__device__ unsigned long long g_tstart[4096], g_tend[4096];
#include "../paper_2604_08812_b200/csrc/kernels.cuh"
using namespace dsel;
#ifndef PROBE_NB
#define PROBE_NB 32
#endif
#ifndef PROBE_MINB
#define PROBE_MINB 1
#endif
int main(int argc, char** argv) {
  int nt = argc > 1 ? atoi(argv[1]) : 128, batch = argc > 2 ? atoi(argv[2]) : 200;
  int mp = ((nt + 7) / 8) * 8; if (mp % 16 == 0 || mp % 16 == 8) mp += 4;
  size_t n2 = (size_t)nt * nt;
  std::vector<double> h(n2 * batch);
  for (int b = 0; b < batch; ++b) for (int i = 0; i < nt; ++i) for (int j = 0; j < nt; ++j)
    h[b * n2 + (size_t)j * nt + i] = (i == j ? nt : 0.0) + 1.0 / (1 + abs(i - j));
  double *src, *L, *gain; int *st, *sc, *sr;
  cudaMalloc(&src, h.size() * 8); cudaMalloc(&L, h.size() * 8); cudaMalloc(&gain, batch * 8);
  cudaMalloc(&st, batch * 4); cudaMalloc(&sc, batch * 4); cudaMalloc(&sr, batch * 4);
  cudaMemcpy(src, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  std::vector<int> cols(batch), rows(batch, 0);
  for (int b = 0; b < batch; ++b) cols[b] = b * nt;  // block b = columns b*nt.., rows 0..nt (ld = nt)
  cudaMemcpy(sc, cols.data(), batch * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(sr, rows.data(), batch * 4, cudaMemcpyHostToDevice);
  CholArgs a{}; a.src = src; a.lds = nt; a.src_col = sc; a.src_row = sr; a.L = L; a.l_stride = n2;
  a.gain = gain; a.status = st; a.nt = nt; a.n = batch; a.mp = mp;
  size_t smem = ((size_t)PROBE_NB * mp + nt) * 8;
  cudaFuncSetAttribute(chol_logdet_kernel<PROBE_NB, PROBE_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) chol_logdet_kernel<PROBE_NB, PROBE_MINB><<<batch, 256, smem>>>(a);
  cudaEventRecord(e0);
  chol_logdet_kernel<PROBE_NB, PROBE_MINB><<<batch, 256, smem>>>(a);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long stamps[128]; cudaMemcpyFromSymbol(stamps, g_stamps, sizeof(stamps));
  double g; cudaMemcpy(&g, gain, 8, cudaMemcpyDeviceToHost);
  printf("nt %d batch %d: %.1f us  gain[0]=%.17g err=%s\n", nt, batch, ms * 1e3, g, cudaGetErrorString(cudaGetLastError()));
  for (int i = 1; i < 128 && stamps[i]; ++i) printf("  stamp %2d: +%lld cycles\n", i, stamps[i] - stamps[i - 1]);
  std::vector<unsigned long long> ts(batch), te(batch);
  cudaMemcpyFromSymbol(ts.data(), g_tstart, batch * 8); cudaMemcpyFromSymbol(te.data(), g_tend, batch * 8);
  unsigned long long mn = ts[0], mx = te[0]; double avg = 0, mxd = 0;
  for (int b = 0; b < batch; ++b) { mn = std::min(mn, ts[b]); mx = std::max(mx, te[b]); avg += te[b] - ts[b]; mxd = std::max(mxd, (double)(te[b] - ts[b])); }
  unsigned long long lastStart = 0; for (int b = 0; b < batch; ++b) lastStart = std::max(lastStart, ts[b] - mn);
  printf("  blocks: span %.1f us, mean block %.1f us, max block %.1f us, last start +%.1f us\n", (mx - mn) / 1e3, avg / batch / 1e3, mxd / 1e3, lastStart / 1e3);
  return 0;
}
