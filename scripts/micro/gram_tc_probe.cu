// Probe of the tcgen05 Gram kernel: one CTA, one stage, known inputs.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I include -I paper_0909_4969_b200/csrc \
//   scripts/micro/gram_tc_probe.cu -o scripts/micro/gram_tc_probe -lcuda
#include "../../paper_0909_4969_b200/csrc/gram_tc.cu"
#include <cstdio>
using namespace machb;
int main(int argc, char** argv) {
    const int mn = argc > 1 ? atoi(argv[1]) : 0;
    if (argc > 3) { uint32_t l = atoi(argv[2]), s_ = atoi(argv[3]); cudaMemcpyToSymbol(g_mn_lbo, &l, 4); cudaMemcpyToSymbol(g_mn_sbo, &s_, 4); printf("lbo %u sbo %u\n", l, s_); }
    Ctx ctx; cudaStreamCreate(&ctx.stream);
    // K-major: dims {32 (inner = K), 256 (R), 1}; MN: dims {256 (R), 32 (K)}
    const int R = 256, K = 32;
    std::vector<float> h(R * K);
    for (int r = 0; r < R; ++r) for (int k = 0; k < K; ++k) {
        float v = (r == k) ? 1.0f : ((r % 7) == (k % 7) ? 0.5f : 0.0f);
        if (mn) h[r + R * k] = v; else h[k + K * r] = v;
    }
    float* x; cudaMalloc(&x, h.size() * 4); cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tm; EncodeTiled enc = encode_fn(); CUresult rc;
    if (mn) {
        const cuuint64_t gdim[2] = {R, K}; const cuuint64_t gs[1] = {R * 4}; const cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
        rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, gdim, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const cuuint64_t gdim[3] = {K, R, 1}; const cuuint64_t gs[2] = {K * 4, (cuuint64_t)K * R * 4}; const cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
        rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, gdim, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("encode rc=%d\n", (int)rc);
    const int ntile = tile_count(R);
    float* part; cudaMalloc(&part, (size_t)ntile * TBM * TBN * 4); cudaMemset(part, 0xff, (size_t)ntile * TBM * TBN * 4);
    unsigned* dbg; cudaMalloc(&dbg, kStageBytes); cudaMemset(dbg, 0, kStageBytes);
    auto kern = mn ? gram_tc_kernel<true> : gram_tc_kernel<false>;
    printf("attr %s\n", cudaGetErrorString(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGramSmem)));
    kern<<<ntile, kGThreads, kGramSmem, ctx.stream>>>(tm, 1, 1, 1, ntile, part, dbg);
    printf("launch %s\n", cudaGetErrorString(cudaGetLastError()));
    printf("sync %s\n", cudaGetErrorString(cudaStreamSynchronize(ctx.stream)));
    std::vector<unsigned> d(kStageBytes / 4); cudaMemcpy(d.data(), dbg, kStageBytes, cudaMemcpyDeviceToHost);
    int nz = 0; for (auto v : d) nz += v != 0;
    printf("stage0 nonzero words %d of %zu; first row words:", nz, d.size());
    for (int i = 0; i < 32; ++i) printf(" %08x", d[i]); printf("\n");
    std::vector<float> p((size_t)ntile * TBM * TBN); cudaMemcpy(p.data(), part, p.size() * 4, cudaMemcpyDeviceToHost);
    // tile 0 = rows 0..127, cols 0..255 (col-major, ld 128)
    double err = 0; int bad = 0;
    for (int t = 0; t < ntile; ++t) { int I, J; tile_of(t, I, J);
      for (int c = 0; c < TBN; ++c) for (int r = 0; r < TBM; ++r) {
        int gr = TBM * I + r, gc = TBN * J + c; if (gr >= R || gc >= R) continue;
        double ref = 0; for (int k = 0; k < K; ++k) ref += (double)h[mn ? gr + R * k : k + K * gr] * h[mn ? gc + R * k : k + K * gc];
        double got = p[(size_t)t * TBM * TBN + (size_t)c * TBM + r];
        if (fabs(got - ref) > 1e-3) { if (bad < 8) printf("  tile %d (%d,%d): got %g ref %g\n", t, gr, gc, got, ref); ++bad; }
      } }
    printf("bad %d\n", bad);
    printf("tile0 row0 cols0..8: "); for (int c = 0; c < 9; ++c) printf("%g ", p[(size_t)c * TBM]); printf("\n");
    return 0;
}
