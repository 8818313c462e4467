"""clock64 timeline for edge_bwd2 (CTA 0, first 32 tiles). on|restore; DSMPNN_TIMELINE=1."""
import shutil, sys
EB = '/root/repo/paper_2402_15106_b200/csrc/edge_bwd2.cuh'
LB = '/root/repo/paper_2402_15106_b200/csrc/layer_bf16_bwd.cu'
if sys.argv[1] == 'restore':
    shutil.copy('/tmp/eb2_clean.cuh', EB); shutil.copy('/tmp/lbb_clean.cu', LB); sys.exit()
shutil.copy(EB, '/tmp/eb2_clean.cuh'); shutil.copy(LB, '/tmp/lbb_clean.cu')
s = open(EB).read()
def rep(a, b):
    global s
    assert a in s, a[:70]
    s = s.replace(a, b, 1)
rep('namespace dsmpnn {\n', 'namespace dsmpnn {\nstatic __device__ unsigned long long *g_tl;\n'
    '#define TL(slot) do { if (g_tl && blockIdx.x == 0 && t < 32) g_tl[t * 32 + (slot)] = clock64(); } while (0)\n')
rep('  const uint32_t tmem = m->tmem;\n', '  const uint32_t tmem = m->tmem;\n  if (g_tl && blockIdx.x == 0 && tid == 0) g_tl[31] = clock64();\n')
LO = 'if (warp == 0 && lane == 0) '
rep('        if (t >= 2) tc::mbar_wait(&m->desc_free[b], ((t >> 1) - 1) & 1);\n',
    f'        {LO}TL(0);\n        if (t >= 2) tc::mbar_wait(&m->desc_free[b], ((t >> 1) - 1) & 1);\n        {LO}TL(1);\n')
rep('        if (t >= 1) tc::mbar_wait(&m->e_empty, (t - 1) & 1);\n', f'        if (t >= 1) tc::mbar_wait(&m->e_empty, (t - 1) & 1);\n        {LO}TL(2);\n')
rep('        tc::mbar_arrive(&m->v_full);\n', '        tc::mbar_arrive(&m->v_full);\n        if (lane == 0) TL(3);\n')
rep("        tc::mbar_wait(&m->a1_ready, t & 1);\n", "        tc::mbar_wait(&m->a1_ready, t & 1);\n        TL(4);\n")
rep('        tc::mma_commit(&m->d2_full);\n', '        tc::mma_commit(&m->d2_full);\n        TL(5);\n')
rep('        tc::mbar_wait(&m->h_ready, p1);  // z2 drained', '        tc::mbar_wait(&m->h_ready, p1);\n        TL(6);  // z2 drained')
rep('        if (t >= 1) tc::mbar_wait(&m->dh_free, (t - 1) & 1);  // U region', '        TL(7);\n        if (t >= 1) tc::mbar_wait(&m->dh_free, (t - 1) & 1);  // U region')
rep('        if (t >= 1) tc::mbar_wait(&m->dh0_free, (t - 1) & 1);  // dH region', '        TL(8);\n        if (t >= 1) tc::mbar_wait(&m->dh0_free, (t - 1) & 1);  // dH region')
rep('        tc::mbar_wait(&m->u_free, p1);  // U drained', '        TL(9);\n        tc::mbar_wait(&m->u_free, p1);  // U drained')
rep('        dsq += tr.nn;\n', '        dsq += tr.nn;\n        TL(10);\n')
EA = 'if (warp == 4 && lane == 0) '
rep('      tc::mbar_wait(&m->d1_full, p1);\n', f'      tc::mbar_wait(&m->d1_full, p1);\n      {EA}TL(11);\n')
rep('        if (cc == 0 && t >= 1) tc::mbar_wait(&m->ah_free, (t - 1) & 1);\n', f'        if (cc == 0 && t >= 1) tc::mbar_wait(&m->ah_free, (t - 1) & 1);\n        if (cc == 0) {{ {EA}TL(12); }}\n')
rep('      tc::mbar_arrive(&m->a1_ready);\n', f'      tc::mbar_arrive(&m->a1_ready);\n      {EA}TL(13);\n')
rep('      tc::mbar_wait(&m->d2_full, p1);\n', f'      tc::mbar_wait(&m->d2_full, p1);\n      {EA}TL(14);\n')
rep('      tc::named_sync(2, 256);\n      tc::tc_fence_after();\n', f'      tc::named_sync(2, 256);\n      {EA}TL(15);\n      tc::tc_fence_after();\n')
rep('      tc::mbar_arrive(&m->h_ready);\n', f'      tc::mbar_arrive(&m->h_ready);\n      {EA}TL(16);\n')
EBG = 'if (warp == 12 && lane == 0) '
rep('      tc::mbar_arrive(&m->mask_read);\n', f'      tc::mbar_arrive(&m->mask_read);\n      {EBG}TL(17);\n')
rep('      tc::mbar_wait(&m->u_full, p1);\n', f'      tc::mbar_wait(&m->u_full, p1);\n      {EBG}TL(18);\n')
rep('      tc::mbar_arrive(&m->u_free);\n', f'      tc::mbar_arrive(&m->u_free);\n      {EBG}TL(19);\n')
rep('        tc::mbar_wait(h == 0 ? &m->dh0_full : &m->dh1_full, p1);\n', f'        tc::mbar_wait(h == 0 ? &m->dh0_full : &m->dh1_full, p1);\n        {EBG}TL(20 + 2 * h);\n')
rep('        tc::mbar_arrive(h == 0 ? &m->dh0_free : &m->dh_free);\n', f'        tc::mbar_arrive(h == 0 ? &m->dh0_free : &m->dh_free);\n        {EBG}TL(21 + 2 * h);\n')
open(EB, 'w').write(s)
l = open(LB).read()
a = '''  kern<<<grid, 512, C::SMEM, s>>>(tW2, tDS, e, v, row_ptr, col, rb, re, eb, ee, pw, b1, b2, b.dS, b.A1, b.dZ2, b.U,
                                  b.db2_part);'''
assert a in l
l = l.replace(a, '''static unsigned long long *dbg = nullptr;
  if (getenv("DSMPNN_TIMELINE") && !dbg) { cudaMalloc(&dbg, 32 * 32 * 8); cudaMemcpyToSymbol(g_tl, &dbg, sizeof(dbg)); }
  if (dbg) cudaMemsetAsync(dbg, 0, 32 * 32 * 8, s);
''' + a + '''
  if (dbg) {
    unsigned long long h[32 * 32];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const char *nm[24] = {"Ld0", "Ld1df", "Ld2ee", "Ld3ve", "M4a1", "M5d2", "M6hr", "M7uf", "M8dh", "M9d0f", "M10end",
                          "A11d1", "A12ah", "A13a1", "A14d2", "A15sy", "A16hr", "B17mr", "B18uf", "B19ua", "B20h0",
                          "B21h0a", "B22h1", "B23h1a"};
    fprintf(stderr, "     ");
    for (int k = 0; k < 24; ++k) fprintf(stderr, "%7s", nm[k]);
    fprintf(stderr, "\\n");
    for (int t = 0; t < 10; ++t) {
      fprintf(stderr, "t%2d: ", t);
      for (int k = 0; k < 24; ++k) fprintf(stderr, "%7lld", h[t * 32 + k] ? (long long)(h[t * 32 + k] - h[31]) : -1LL);
      fprintf(stderr, "\\n");
    }
  }''')
open(LB, 'w').write(l)
