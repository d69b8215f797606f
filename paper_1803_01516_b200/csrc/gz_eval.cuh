// gz_eval.cuh -- accuracy accounting and penalty sweeps on the device
// (SURVEY.md §8(f) items 2-3).  Included at the end of gz_solver.cu.
//
//  * gz_ground_truth_to_depth  imaging.py:155-201: ground-truth disparity image
//    -> per-site depth numbers (nearest surface wins), valid mask, counters.
//  * gz_error_count            evalreport.py:47-61: total |label - depth| over
//    valid sites, evaluated count, histogram with a pooled tail bucket.
//  * gz_solve_volume_batch     evalreport.py:88-126 (sweep_penalty's solves):
//    one volume, n energy parameter sets, up to 8 exact solves in flight, each
//    a cooperative launch on 1/8 of the SMs with its own workspace slice; the
//    labelings stay on the device for gz_error_count.

namespace {

// geometry.py:37-47 round_away_half: halve, .5 away from zero
__device__ __forceinline__ long long round_away_half(long long a) {
    return a >= 0 ? (a + 1) / 2 : -((-a + 1) / 2);
}

// One thread per pixel: imaging.py:172-190 (best = min depth number per site).
__global__ void k_gt_scatter(const uint8_t *__restrict__ gt, int h, int w, int scale, gz_gaze g, int32_t *best,
                             unsigned long long *cnt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long off = 0, oor = 0, keep = 0;
    if (i < (long long)h * w) {
        const int v = gt[i];
        if (v) {
            const long long ys = i / w, xs = i - ys * w;
            const long long dis = ((long long)v * 2 + scale) / (2 * scale);   // round half up
            const long long W = xs - round_away_half(g.lw_offset + g.rw_offset) + round_away_half(dis);
            const long long S = round_away_half(g.lw_offset - g.rw_offset) - round_away_half(dis);
            const long long gi = (W - g.offset1) - g.g_min;
            const long long yi = (ys - g.h_offset + g.offset2) - g.y_min;
            const long long k = (S - g.offset3) - g.d_min;
            const bool on_grid = gi >= 0 && gi < g.cols && yi >= 0 && yi < g.rows;
            const bool in_range = k >= 0 && k < g.m;
            if (!on_grid) off = 1;
            else if (!in_range) oor = 1;
            else {
                keep = 1;
                atomicMin(&best[yi * g.cols + gi], (int32_t)k);
            }
        }
    }
    warp_add_u64(&cnt[0], (long long)oor);
    warp_add_u64(&cnt[1], (long long)off);
    warp_add_u64(&cnt[2], (long long)keep);
}

// imaging.py:191-194: valid = best < sentinel, depth = valid ? best : 0
__global__ void k_gt_finish(int32_t *depth, uint8_t *valid, int P, int m, unsigned long long *cnt) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nv = 0;
    if (c < P) {
        const int b = depth[c];
        const bool ok = b < m;
        valid[c] = ok ? 1 : 0;
        depth[c] = ok ? b : 0;
        nv = ok ? 1 : 0;
    }
    warp_add_u64(&cnt[3], (long long)nv);
}

// evalreport.py:47-61 over `batch` labelings against one ground truth:
// out[b * (tail + 3)] = total error, [+1] evaluated, [+2 ..] histogram[0..tail].
// Block-level shared histogram, one atomic per bucket per block.
__global__ void k_error_count(const int32_t *__restrict__ lab, const int32_t *__restrict__ depth,
                              const uint8_t *__restrict__ valid, int P, int tail, unsigned long long *out) {
    extern __shared__ unsigned long long s_h[];   // tail + 3 words
    const int b = blockIdx.y;
    for (int i = threadIdx.x; i < tail + 3; i += blockDim.x) s_h[i] = 0ull;
    __syncthreads();
    const int32_t *L = lab + (size_t)b * P;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < P; c += gridDim.x * blockDim.x) {
        if (!valid[c]) continue;
        const long long d = llabs((long long)L[c] - (long long)depth[c]);
        atomicAdd(&s_h[0], (unsigned long long)d);
        atomicAdd(&s_h[1], 1ull);
        atomicAdd(&s_h[2 + (d < tail ? d : tail)], 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < tail + 3; i += blockDim.x)
        if (s_h[i]) atomicAdd(&out[(size_t)b * (tail + 3) + i], s_h[i]);
}

// imaging.py:228-246 write_disparity_image: each site paints its right-image
// pixel x = g + d with dis * scale, the nearer (larger disparity) wins.
__global__ void k_render_disparity(const int32_t *__restrict__ lab, gz_gaze g, int img_w, int img_h, int scale,
                                   int32_t *img) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.rows * g.cols) return;
    const int yy = c / g.cols, gg = c - yy * g.cols;
    const long long d = (long long)g.d_min + lab[c];
    const long long dis = (long long)(img_w - 1) - 2 * d;
    const long long x = (long long)g.g_min + gg + d, y = (long long)g.y_min + yy;
    if (x < 0 || x >= img_w || y < 0 || y >= img_h) return;
    atomicMax(&img[y * img_w + x], (int32_t)(dis * scale));
}

__global__ void k_i32_to_u8(const int32_t *__restrict__ src, uint8_t *dst, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (uint8_t)src[i];
}

}  // namespace

extern "C" {

int gz_render_disparity(const int32_t *labels, const gz_gaze *gaze, int32_t img_w, int32_t img_h, int32_t scale,
                        int32_t *scratch, uint8_t *image_out, void *stream) {
    if (!labels || !gaze || !scratch || !image_out || img_w < 1 || img_h < 1 || scale < 1) return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = (long long)img_w * img_h;
    const int P = gaze->rows * gaze->cols;
    CK(cudaMemsetAsync(scratch, 0, (size_t)n * 4, s));
    k_render_disparity<<<(P + 255) / 256, 256, 0, s>>>(labels, *gaze, img_w, img_h, scale, scratch);
    k_i32_to_u8<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scratch, image_out, n);
    CK(cudaGetLastError());
    return GZ_OK;
}


int gz_ground_truth_to_depth(const uint8_t *gt, int32_t img_h, int32_t img_w, int32_t scale, const gz_gaze *gaze,
                             int32_t *depth_out, uint8_t *valid_out, int64_t *counts_out, void *stream) {
    if (!gt || !gaze || !depth_out || !valid_out || !counts_out || img_h < 1 || img_w < 1 || scale < 1) return GZ_ERR_ARG;
    if (gaze->rows < 1 || gaze->cols < 1 || gaze->m < 1) return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int P = gaze->rows * gaze->cols;
    unsigned long long *cnt = (unsigned long long *)counts_out;   // [0] out_of_range [1] off_grid [2] kept [3] valid
    CK(cudaMemsetAsync(cnt, 0, 4 * 8, s));
    k_fill_i32<<<(P + 255) / 256, 256, 0, s>>>(depth_out, P, gaze->m);   // sentinel: any real label is smaller
    const long long n = (long long)img_h * img_w;
    k_gt_scatter<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(gt, img_h, img_w, scale, *gaze, depth_out, cnt);
    k_gt_finish<<<(P + 255) / 256, 256, 0, s>>>(depth_out, valid_out, P, gaze->m, cnt);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_error_count(const int32_t *labels, int32_t batch, const int32_t *depth, const uint8_t *valid, int32_t rows,
                   int32_t cols, int32_t tail, int64_t *out, void *stream) {
    if (!labels || !depth || !valid || !out || batch < 1 || rows < 1 || cols < 1 || tail < 1 || tail > 4096)
        return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int P = rows * cols;
    CK(cudaMemsetAsync(out, 0, (size_t)batch * (tail + 3) * 8, s));
    int blocks = (P + 255) / 256;
    if (blocks > 296) blocks = 296;
    k_error_count<<<dim3(blocks, batch), 256, (tail + 3) * 8, s>>>(labels, depth, valid, P, tail,
                                                                    (unsigned long long *)out);
    CK(cudaGetLastError());
    return GZ_OK;
}

int gz_solve_volume_batch(const int32_t *vol, int32_t rows, int32_t cols, int32_t m, const gz_energy *energies,
                          int32_t n, const gz_sched *sched, int32_t *labels_out, gz_stats *stats_out, void *workspace,
                          size_t workspace_bytes, void *stream) {
    if (!vol || !energies || !labels_out || n < 1 || rows < 1 || cols < 1 || m < 2) return GZ_ERR_ARG;
    for (int b = 0; b < n; ++b)
        if (energies[b].penalty < 0 || energies[b].inhibit < 0) return GZ_ERR_ARG;
    if (!index_fits(rows, cols, m)) return GZ_ERR_OVERFLOW;
    const int P = rows * cols;
    const size_t one = ws_bytes(rows, cols, m);
    if (workspace_bytes < one) return GZ_ERR_WORKSPACE;
    int rc = check_sm100();
    if (rc) return rc;
    if (choose_solver(m, sched) != 4 || (sched && (sched->flags & GZ_SCHED_CAPPED))) return GZ_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    // census (full windows: source capacity = sum of the first chain arcs, the
    // same for every penalty; hard mode counts no uncuttable source arcs)
    Workspace w0 = carve(workspace, rows, cols, m);
    CK(cudaMemsetAsync(w0.ctr, 0, 24, s));
    gz_energy e0 = energies[0];
    k_source_caps<<<(P + 255) / 256, 256, 0, s>>>(vol, rows, cols, m, nullptr, nullptr, e0, w0.ctr);
    unsigned long long census[3];
    CK(cudaMemcpyAsync(census, w0.ctr, 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (census[0] >= 0x7fffffffull) return GZ_ERR_OVERFLOW;
    int hcap_hard = 1 << 16;
    while ((unsigned long long)hcap_hard <= census[0]) hcap_hard <<= 1;
    if ((unsigned long long)hcap_hard + census[0] >= 0x7fffffffull) hcap_hard = 0;
    int conc = 8;
    if (const char *cs = getenv("GZ_PAIR_CONC")) conc = atoi(cs);
    if (conc > DevicePool::MAX_STREAMS) conc = DevicePool::MAX_STREAMS;
    if ((size_t)conc * one > workspace_bytes) conc = (int)(workspace_bytes / one);
    if (conc > n) conc = n;
    if (conc < 1) conc = 1;
    DevicePool *pool = device_pool();
    if (!pool) return GZ_ERR_CUDA;
    std::lock_guard<std::mutex> lock(pool->mu);
    if ((rc = pool->streams_ready())) return rc;
    if ((rc = pool->pinned_ready((size_t)n * gz::CTR_COUNT))) return rc;
    cudaStream_t *streams = pool->streams;
    unsigned long long *pinned = pool->pinned;
    cudaEvent_t fork;
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventRecord(fork, s));
    for (int k = 0; k < conc; ++k) CK(cudaStreamWaitEvent(streams[k], fork, 0));
    Pending *pend = new Pending[n];
    const int lp = lanes_for(m);
    for (int b = 0; b < n && rc == GZ_OK; ++b) {
        const int k = b % conc;
        Workspace w = carve((uint8_t *)workspace + (size_t)k * one, rows, cols, m);
        const long long nel = (long long)P * lp;
        k_to_colmajor<<<(unsigned)((nel + 255) / 256), 256, 0, streams[k]>>>(vol, P, m, lp, w.vol);
        if (cudaGetLastError() != cudaSuccess) { rc = GZ_ERR_CUDA; break; }
        const int hcap = energies[b].hard_inhibit ? hcap_hard : HARD_CAP_DEFAULT;
        if (hcap == 0) { rc = GZ_ERR_OVERFLOW; break; }
        rc = solve_launch(w, rows, cols, m, &energies[b], sched, nullptr, nullptr, labels_out + (size_t)b * P,
                          streams[k], hcap, conc, pinned + (size_t)b * gz::CTR_COUNT, &pend[b]);
    }
    for (int k = 0; k < conc; ++k) {
        cudaEvent_t join;
        cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
        cudaEventRecord(join, streams[k]);
        cudaStreamWaitEvent(s, join, 0);
        cudaEventDestroy(join);
    }
    cudaEventDestroy(fork);
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == GZ_OK) rc = GZ_ERR_CUDA;
    for (int b = 0; b < n; ++b) {
        if (!pend[b].e0) continue;
        const int r = solve_finish(pend[b], stats_out ? stats_out + b : nullptr);
        if (rc == GZ_OK) rc = r;
    }
    delete[] pend;
    if (rc) return rc;
    if (stats_out)
        for (int b = 0; b < n; ++b)
            if (stats_out[b].energy != stats_out[b].labeling_energy) return GZ_ERR_CONSISTENCY;
    return GZ_OK;
}

}  // extern "C"
