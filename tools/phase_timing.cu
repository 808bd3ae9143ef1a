// Phase timing harness for the column passes (debug tool, not the product).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DVX_PHASE_TIMING
//        -I include -I paper_2407_02363_b200/csrc tools/phase_timing.cu -o tools/phase_timing
// Run:   tools/phase_timing occ.raw nx ny nz   (occ.raw: uint8 C-order occupancy)
#include "../paper_2407_02363_b200/csrc/vx_edt.cu"

#include <cstdio>
#include <vector>

int main(int argc, char **argv) {
    if (argc < 5) { fprintf(stderr, "usage: %s occ.raw nx ny nz\n", argv[0]); return 2; }
    const int nx = atoi(argv[2]), ny = atoi(argv[3]), nz = atoi(argv[4]);
    const size_t n = (size_t)nx * ny * nz;
    std::vector<uint8_t> h(n);
    FILE *f = fopen(argv[1], "rb");
    if (!f || fread(h.data(), 1, n, f) != n) { fprintf(stderr, "read failed\n"); return 1; }
    fclose(f);
    vx::EdtPlan p;
    vx::make_plan(nx, ny, nz, &p, 0);
    uint8_t *occ; int32_t *site; void *scratch; unsigned long long *buf;
    cudaMalloc(&occ, n); cudaMalloc(&site, n * 4);
    cudaMalloc(&scratch, vx::scratch_bytes_for(p, 1));
    const long long tiles = (long long)((nz + 31) / 32) * std::max(nx, ny);
    cudaMalloc(&buf, tiles * 8 * 8);
    cudaMemcpy(occ, h.data(), n, cudaMemcpyHostToDevice);
    int32_t *s1 = (int32_t *)scratch;
    const size_t s1b = (n * 4 + 255) & ~(size_t)255;
    void *s2 = (char *)scratch + s1b;
    const size_t s2b = (n * 4 + 255) & ~(size_t)255;
    const bool sparse = vx::sparse_ok(p, 1);
    const vx::SparseRows sp = vx::sparse_rows_at((char *)scratch + s1b + s2b + p.gstack_bytes, p);
    const vx::SparseRows *spp = sparse ? &sp : nullptr;
    if (sparse) { vx::launch_slice_list(occ, p, sp, 0); cudaDeviceSynchronize(); }
    printf("sparse path: %d\n", (int)sparse);
    {   // plain kernel timings (CUDA events), instrumentation buffer detached
        unsigned long long *null_buf = nullptr;
        cudaMemcpyToSymbol(vx::g_phase_buf, &null_buf, sizeof null_buf);
        cudaEvent_t e[4];
        for (auto &x : e) cudaEventCreate(&x);
        float t1 = 0, t2 = 0, t3 = 0;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(e[0]);
            vx::launch_pass1(occ, s1, nx, ny, nz, 0, spp);
            cudaEventRecord(e[1]);
            vx::launch_pass2(s1, s2, nullptr, p, nx, 0, spp);
            cudaEventRecord(e[2]);
            vx::launch_pass3(s2, site, s1, p, 1, 0, ny, 0, spp);
            cudaEventRecord(e[3]);
            cudaEventSynchronize(e[3]);
            float a, b, c;
            cudaEventElapsedTime(&a, e[0], e[1]);
            cudaEventElapsedTime(&b, e[1], e[2]);
            cudaEventElapsedTime(&c, e[2], e[3]);
            if (rep >= 2) { t1 += a / 4; t2 += b / 4; t3 += c / 4; }
        }
        printf("kernel ms: pass1 %.4f pass2 %.4f pass3 %.4f  total %.4f\n", t1, t2, t3, t1 + t2 + t3);
        cudaMemcpyToSymbol(vx::g_phase_buf, &buf, sizeof buf);
    }
    for (int pass = 2; pass <= 3; ++pass) {
        for (int rep = 0; rep < 3; ++rep) {
            vx::launch_pass1(occ, s1, nx, ny, nz, 0, spp);
            vx::launch_pass2(s1, s2, nullptr, p, nx, 0, spp);
            if (pass == 3) {
                cudaMemset(buf, 0, tiles * 64);
                vx::launch_pass3(s2, site, s1, p, 1, 0, ny, 0, spp);
            }
            cudaDeviceSynchronize();
        }
        if (pass == 2) {  // re-run pass 2 with the buffer cleared
            cudaMemset(buf, 0, tiles * 64);
            vx::launch_pass2(s1, s2, nullptr, p, nx, 0, spp);
            cudaDeviceSynchronize();
        }
        const long long nt = (long long)((nz + 31) / 32) * (pass == 2 ? nx : ny);
        std::vector<unsigned long long> t(nt * 8);
        cudaMemcpy(t.data(), buf, nt * 64, cudaMemcpyDeviceToHost);
        double acc[7] = {0};
        long long cnt = 0;
        for (long long i = 0; i < nt; ++i) {
            if (!t[i * 8 + 6]) continue;
            ++cnt;
            for (int q = 0; q < 6; ++q) acc[q] += (double)(t[i * 8 + q + 1] - t[i * 8 + q]);
            acc[6] += (double)(t[i * 8 + 6] - t[i * 8]);
        }
        if (pass == 3 && getenv("VX_HULL_HIST")) {   // hull-size histogram (k_pass3_stream slot 7)
            long long hist[9] = {0};
            for (long long i = 0; i < nt; ++i) {
                const unsigned long long h = t[i * 8 + 7];
                int b = 0;
                while (b < 8 && (1ull << (b + 1)) <= h) ++b;
                hist[b]++;
            }
            printf("hull max per tile histogram (<2,<4,..,>=256):");
            for (int b = 0; b < 9; ++b) printf(" %lld", hist[b]);
            printf("\n");
        }
        printf("pass %d: %lld tiles; mean cycles: tma_wait %.0f  phaseA %.0f  merges %.0f  phaseC %.0f  "
               "phaseD(warp0) %.0f  tail %.0f  total %.0f\n", pass, cnt, acc[0] / cnt, acc[1] / cnt,
               acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt, acc[6] / cnt);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
