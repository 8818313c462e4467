"""clock64 timeline for edge_fwd2 (CTA 0, first 32 tiles). on|restore; DSMPNN_TIMELINE=1."""
import shutil, sys
EF = '/root/repo/paper_2402_15106_b200/csrc/edge_fwd2.cuh'
LB = '/root/repo/paper_2402_15106_b200/csrc/layer_bf16.cu'
if sys.argv[1] == 'restore':
    shutil.copy('/tmp/ef2_clean2.cuh', EF); shutil.copy('/tmp/lb_clean2.cu', LB); sys.exit()
shutil.copy(EF, '/tmp/ef2_clean2.cuh'); shutil.copy(LB, '/tmp/lb_clean2.cu')
s = open(EF).read()
def rep(a, b):
    global s
    assert a in s, a[:70]
    s = s.replace(a, b, 1)
rep('namespace dsmpnn {\n', 'namespace dsmpnn {\nstatic __device__ unsigned long long *g_tlf;\n'
    '#define TL(slot) do { if (g_tlf && blockIdx.x == 0 && t < 32) g_tlf[t * 32 + (slot)] = clock64(); } while (0)\n')
rep('  const uint32_t tmem = m->tmem;\n', '  const uint32_t tmem = m->tmem;\n  if (g_tlf && blockIdx.x == 0 && tid == 0) g_tlf[31] = clock64();\n')
EA = 'if (warp == 4 && lane == 0) '
rep('      tc::mbar_wait(&m->d1_full[b], ph);\n', f'      tc::mbar_wait(&m->d1_full[b], ph);\n      {EA}TL(0);\n')
rep('        if (jj == 0 && t >= 1) tc::mbar_wait(&m->ah_free, (t - 1) & 1);\n',
    f'        if (jj == 0 && t >= 1) tc::mbar_wait(&m->ah_free, (t - 1) & 1);\n        if (jj == 0) {{ {EA}TL(1); }}\n')
rep('      tc::mbar_wait(&m->d2_full[0], p1);\n', f'      {EA}TL(2);\n      tc::mbar_wait(&m->d2_full[0], p1);\n      {EA}TL(3);\n')
rep('      tc::mbar_wait(&m->d2_full[1], p1);\n', f'      tc::mbar_wait(&m->d2_full[1], p1);\n      {EA}TL(4);\n')
rep('      tc::mbar_arrive(&m->h_ready[1]);\n', f'      tc::mbar_arrive(&m->h_ready[1]);\n      {EA}TL(5);\n')
rep('        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);\n        if (!m->desc[b].more) return false;\n',
    '        tc::mbar_wait(&m->e_full[b], (t >> 1) & 1);\n        TL(6);\n        if (!m->desc[b].more) return false;\n')
rep('        tc::mma_bf16_ss(tmem + b * 256, tc::sdesc(aE', '        TL(7);\n        tc::mma_bf16_ss(tmem + b * 256, tc::sdesc(aE')
rep("        const uint32_t r = tmem + b * 256;\n", "        const uint32_t r = tmem + b * 256;\n        TL(8);\n")
rep('        tc::mbar_wait(&m->v_full, p1);\n', '        tc::mbar_wait(&m->v_full, p1);\n        TL(9);\n')
rep('        tc::mma_commit(&m->s_full);\n', '        TL(10);\n        tc::mma_commit(&m->s_full);\n')
LO = 'if (li == 0) '
rep('      if (t >= 2) tc::mbar_wait(&m->desc_free[b], ((t >> 1) - 1) & 1);\n',
    f'      if (t >= 2) tc::mbar_wait(&m->desc_free[b], ((t >> 1) - 1) & 1);\n      {LO}TL(11);\n')
rep('      if (t >= 1) tc::mbar_wait(&m->e_empty, (t - 1) & 1);\n', f'      if (t >= 1) tc::mbar_wait(&m->e_empty, (t - 1) & 1);\n      {LO}TL(12);\n')
rep('      if (t >= 1) tc::mbar_wait(&m->v_empty, (t - 1) & 1);\n', f'      if (t >= 1) tc::mbar_wait(&m->v_empty, (t - 1) & 1);\n      {LO}TL(13);\n')
EB = 'if (warp == 12 && lane == 0) '
rep('      tc::mbar_wait(&m->s_full, p1);\n', f'      tc::mbar_wait(&m->s_full, p1);\n      {EB}TL(14);\n')
rep('      if (lane == 0) tc::mbar_arrive(&m->region_free[b]);\n', f'      if (lane == 0) tc::mbar_arrive(&m->region_free[b]);\n      {EB}TL(15);\n')
open(EF, 'w').write(s)
l = open(LB).read()
import re
m = re.search(r'  kern<<<grid, 512, C::SMEM, s>>>\([^;]*;\n', l)
a = m.group(0)
l = l.replace(a, '''  static unsigned long long *dbg = nullptr;
  if (getenv("DSMPNN_TIMELINE") && !dbg) { cudaMalloc(&dbg, 32 * 32 * 8); cudaMemcpyToSymbol(g_tlf, &dbg, sizeof(dbg)); }
  if (dbg) cudaMemsetAsync(dbg, 0, 32 * 32 * 8, s);
''' + a + '''  if (dbg) {
    unsigned long long h[32 * 32];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const char *nm[16] = {"A0d1", "A1ahf", "A2a1", "A3d2a", "A4d2b", "A5h", "M6ef", "M7rf", "M8nx", "M9vf", "M10sf",
                          "L11df", "L12ee", "L13ve", "B14sf", "B15rf"};
    fprintf(stderr, "     ");
    for (int k = 0; k < 16; ++k) fprintf(stderr, "%7s", nm[k]);
    fprintf(stderr, "\\n");
    for (int t = 0; t < 10; ++t) {
      fprintf(stderr, "t%2d: ", t);
      for (int k = 0; k < 16; ++k) fprintf(stderr, "%7lld", h[t * 32 + k] ? (long long)(h[t * 32 + k] - h[31]) : -1LL);
      fprintf(stderr, "\\n");
    }
  }
''')
open(LB, 'w').write(l)
