// gz_bands.cuh -- one problem solved as row bands over several GPUs (SURVEY.md
// §8(e), BASELINE config 5: 3840x2160x256 across 8 B200).  Included at the end
// of gz_solver.cu (same translation unit: Workspace, carve, solve_launch).
//
// The B200 shape of the reference's "halo exchange": there is none as a
// separate step.  Every state plane of the v4 solver ([site][LPT] int32 planes,
// [word][site] bit planes) is ONE virtual address range (CUDA VMM); band k's
// site rows of every plane are backed by physical memory on devices[k], and
// every device maps the whole range.  Band k runs as a cooperative launch on
// devices[k] over its own tile rows, site range and pulse groups
// (gz_tilesolve.cuh: Geo), and all launches form ONE team: one barrier word
// (system-scope fences when the bands span GPUs).  Arc pairs, heights and
// inbox words across a band edge are read and written in place over NVLink
// (peer loads, stores and atomics), overlapped with the band's own work;
// only the edge rows' traffic crosses the link (~10 MB per edge per sweep at
// C5, against ~12 GB of band-local pass traffic).
//
// Because placement affects only speed, the same code runs with several bands
// on ONE device (devices = {0, 0, ...}: the bands split its SMs), which is how
// the band logic is tested on a single GPU.

#include <cudaTypedefs.h>

#include <vector>

namespace {

struct VmmApi {
    PFN_cuMemCreate create = nullptr;
    PFN_cuMemRelease release = nullptr;
    PFN_cuMemAddressReserve reserve = nullptr;
    PFN_cuMemAddressFree addr_free = nullptr;
    PFN_cuMemMap map = nullptr;
    PFN_cuMemUnmap unmap = nullptr;
    PFN_cuMemSetAccess set_access = nullptr;
    PFN_cuMemGetAllocationGranularity granularity = nullptr;
};

// Driver entry points through the runtime (no link-time libcuda dependency, so
// the library still loads on a host without a driver).
int vmm_api(VmmApi &v) {
    static VmmApi cached;
    static bool have = false;
    if (have) { v = cached; return GZ_OK; }
    cudaDriverEntryPointQueryResult q;
#define GZ_DRV(field, name)                                                                        \
    if (cudaGetDriverEntryPoint(name, (void **)&cached.field, cudaEnableDefault, &q) != cudaSuccess || \
        q != cudaDriverEntryPointSuccess || !cached.field)                                         \
        return GZ_ERR_CUDA;
    GZ_DRV(create, "cuMemCreate")
    GZ_DRV(release, "cuMemRelease")
    GZ_DRV(reserve, "cuMemAddressReserve")
    GZ_DRV(addr_free, "cuMemAddressFree")
    GZ_DRV(map, "cuMemMap")
    GZ_DRV(unmap, "cuMemUnmap")
    GZ_DRV(set_access, "cuMemSetAccess")
    GZ_DRV(granularity, "cuMemGetAllocationGranularity")
#undef GZ_DRV
    have = true;
    v = cached;
    return GZ_OK;
}

// A byte range of the workspace whose contents are indexed by site: byte o
// belongs to site ((o - off) % period) / bps.
struct SiteRegion {
    size_t off, len, period, bps;
};

// One virtual range; physical backing placed per 2 MB chunk on the device of
// the band that owns the chunk's sites.
struct BandMemory {
    VmmApi api;
    CUdeviceptr base = 0;
    size_t size = 0;
    std::vector<CUmemGenericAllocationHandle> handles;

    // site_band: band of every site; band_dev: device of every band.  One
    // physical allocation per run of chunks with one owner band (bands on one
    // device are still separate allocations, so a forced multi-device run on
    // one GPU exercises the same placement as a real one).
    int alloc(size_t bytes, const std::vector<SiteRegion> &regions, const std::vector<int> &site_band,
              const std::vector<int> &band_dev, int home, const std::vector<int> &devices) {
        int rc = vmm_api(api);
        if (rc) return rc;
        size_t gran = 0;
        for (int d : devices) {
            CUmemAllocationProp pr = {};
            pr.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            pr.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            pr.location.id = d;
            size_t g = 0;
            if (api.granularity(&g, &pr, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) return GZ_ERR_CUDA;
            if (g > gran) gran = g;
        }
        size = (bytes + gran - 1) / gran * gran;
        if (api.reserve(&base, size, gran, 0, 0) != CUDA_SUCCESS) { base = 0; return GZ_ERR_CUDA; }
        const size_t nchunks = size / gran;
        auto owner = [&](size_t o) {   // owning band, -1: the home device's
            for (const SiteRegion &r : regions)
                if (o >= r.off && o < r.off + r.len) {
                    const size_t site = ((o - r.off) % r.period) / r.bps;
                    if (site < site_band.size()) return site_band[site];
                }
            return -1;
        };
        size_t c = 0;
        while (c < nchunks) {   // runs of chunks with one owner -> one physical allocation each
            const int ob = owner(c * gran + gran / 2);
            const int d = ob < 0 ? home : band_dev[ob];
            size_t e = c + 1;
            while (e < nchunks && owner(e * gran + gran / 2) == ob) ++e;
            CUmemAllocationProp pr = {};
            pr.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            pr.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            pr.location.id = d;
            CUmemGenericAllocationHandle h;
            if (api.create(&h, (e - c) * gran, &pr, 0) != CUDA_SUCCESS) return GZ_ERR_CUDA;
            handles.push_back(h);
            if (api.map(base + c * gran, (e - c) * gran, 0, h, 0) != CUDA_SUCCESS) return GZ_ERR_CUDA;
            c = e;
        }
        std::vector<CUmemAccessDesc> acc;
        for (int d : devices) {
            bool seen = false;
            for (const CUmemAccessDesc &a : acc) seen |= a.location.id == d;
            if (seen) continue;
            CUmemAccessDesc a = {};
            a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            a.location.id = d;
            a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            acc.push_back(a);
        }
        if (api.set_access(base, size, acc.data(), acc.size()) != CUDA_SUCCESS) return GZ_ERR_CUDA;
        return GZ_OK;
    }
    ~BandMemory() {
        if (!base) return;
        api.unmap(base, size);
        for (CUmemGenericAllocationHandle h : handles) api.release(h);
        api.addr_free(base, size);
    }
};

// Everything gz_solve_volume_banded creates besides the VMM range, released on
// every return path: the streams are drained before the memory goes, the
// staging buffer is freed and the caller's current device is restored.
struct BandsCleanup {
    int prev_dev = 0, home = 0, n = 0;
    const int32_t *devices = nullptr;
    cudaStream_t *band_streams = nullptr;
    cudaStream_t s = nullptr;
    int32_t *stage = nullptr;
    ~BandsCleanup() {
        for (int k = 0; k < n; ++k)
            if (band_streams[k]) {
                cudaSetDevice(devices[k]);
                cudaStreamSynchronize(band_streams[k]);
                cudaStreamDestroy(band_streams[k]);
            }
        cudaSetDevice(home);
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
        if (stage) cudaFree(stage);
        cudaSetDevice(prev_dev);
    }
};

}  // namespace

extern "C" {

int gz_solve_volume_banded(const int32_t *vol_host, int32_t rows, int32_t cols, int32_t m, const gz_energy *energy,
                           const gz_sched *sched, const int32_t *lo_host, const int32_t *hi_host, int32_t nbands,
                           const int32_t *devices, int32_t *labels_host, gz_stats *stats_out) {
    if (!vol_host || !energy || !devices || !labels_host || rows < 1 || cols < 1 || m < 2 ||
        (!lo_host) != (!hi_host) || nbands < 1 || nbands > MAX_BANDS)
        return GZ_ERR_ARG;
    if (energy->penalty < 0 || energy->inhibit < 0) return GZ_ERR_ARG;
    if (!index_fits(rows, cols, m)) return GZ_ERR_OVERFLOW;
    if (choose_solver(m, sched) != 4 || (sched && (sched->flags & GZ_SCHED_CAPPED))) return GZ_ERR_ARG;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int k = 0; k < nbands; ++k)
        if (devices[k] < 0 || devices[k] >= ndev) return GZ_ERR_ARG;
    BandPlan bp;
    for (int k = 0; k < MAX_BANDS; ++k) bp.stream[k] = nullptr;
    bp.n = nbands;
    bp.home = devices[0];
    // GZ_FORCE_SYS=1: run the multi-device code path even when every band is on
    // one GPU -- system-scope fences and atomics in the team barrier and on
    // cross-band state, one physical allocation per band -- so the single-GPU
    // box executes what an 8-GPU band solve executes
    const char *fs = getenv("GZ_FORCE_SYS");
    const bool force_sys = fs && atoi(fs) != 0;
    std::vector<int> devs(devices, devices + nbands);
    BandMemory mem;       // declared before the cleanup: released after the streams are drained
    BandsCleanup cl;
    CK(cudaGetDevice(&cl.prev_dev));
    cl.home = bp.home;
    cl.n = nbands;
    cl.devices = devices;
    cl.band_streams = bp.stream;
    for (int k = 0; k < nbands; ++k) {
        bp.dev[k] = devices[k];
        bp.multi_dev |= devices[k] != devices[0];
        CK(cudaSetDevice(devices[k]));
        int rc = check_sm100();
        if (rc) return rc;
    }
    if (force_sys && nbands > 1) bp.multi_dev = 1;
    if (const char *sp = getenv("GZ_BAND_SPIN_MS")) bp.spin_ms = atoi(sp);
    // team: one CTA per SM (the v4 instances run at occupancy 1 for lone solves),
    // the SMs of a device split evenly between the bands it hosts
    int nb = 0;
    for (int k = 0; k < nbands; ++k) {
        int sms = 0, share = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, devices[k]));
        for (int j = 0; j < nbands; ++j) share += devices[j] == devices[k];
        bp.grid[k] = sms / share;
        if (bp.grid[k] < 1) return GZ_ERR_ARG;
        nb += bp.grid[k];
    }
    const int P = rows * cols, NW = words_for(m);
    bp.geo = tile_geo(rows, cols, nb, NW, 1);
    if (bp.geo.ny < nbands) return GZ_ERR_ARG;   // fewer tile rows than bands
    std::vector<int> site_band((size_t)P, 0);
    for (int k = 0; k < nbands; ++k) {
        const gz4::Geo gk = band_geo(bp.geo, rows, cols, nbands, k, 0, 0, 0);
        for (int c = gk.c0; c < gk.c1; ++c) site_band[(size_t)c] = k;
    }
    std::vector<int> band_dev(devs);
    // workspace layout (carve) as site-indexed regions, plus lo/hi columns
    const size_t wsb = ws_bytes(rows, cols, m), colb = align_up((size_t)P * 4);
    const size_t total = wsb + 2 * colb + 512;
    std::vector<SiteRegion> regions;
    {
        Workspace f = carve((void *)(uintptr_t)0x100000000ull, rows, cols, m);
        const size_t b0 = 0x100000000ull;
        const int mp = m > lanes_for(m) ? m : lanes_for(m);
        const size_t plane = align_up((size_t)mp * P * 4);
        regions.push_back({(size_t)((uintptr_t)f.vol - b0), 12 * plane, plane, (size_t)mp * 4});
        regions.push_back({(size_t)((uintptr_t)f.reach - b0), 3 * colb, colb, 4});
        regions.push_back({(size_t)((uintptr_t)f.bits.mask - b0), (size_t)22 * NW * P * 4, (size_t)P * 4, 4});
        regions.push_back({(size_t)((uintptr_t)f.bits.R0 - b0), 3 * colb, colb, 4});
        regions.push_back({wsb + 256, 2 * colb, colb, 4});
    }
    if (!force_sys) {   // runs split by device only: map every band to its device's first band
        for (size_t c = 0; c < site_band.size(); ++c) {
            const int d = devs[site_band[c]];
            for (int j = 0; j < nbands; ++j)
                if (devs[j] == d) { site_band[c] = j; break; }
        }
    }
    CK(cudaSetDevice(bp.home));
    int rc = mem.alloc(total, regions, site_band, band_dev, bp.home, devs);
    if (rc) return rc;
    uint8_t *base = (uint8_t *)(uintptr_t)mem.base;
    Workspace w = carve(base, rows, cols, m);
    int32_t *lo = nullptr, *hi = nullptr;
    CK(cudaStreamCreateWithFlags(&cl.s, cudaStreamNonBlocking));
    cudaStream_t s = cl.s;
    if (lo_host) {
        lo = (int32_t *)(base + wsb + 256);
        hi = (int32_t *)((uint8_t *)lo + colb);
        CK(cudaMemcpyAsync(lo, lo_host, (size_t)P * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(hi, hi_host, (size_t)P * 4, cudaMemcpyHostToDevice, s));
    }
    // data term: staged once on the home device in (rows, cols, m) order, census,
    // then scattered into the banded solver layout (remote bands over NVLink)
    CK(cudaMalloc((void **)&cl.stage, (size_t)P * m * 4));
    CK(cudaMemcpyAsync(cl.stage, vol_host, (size_t)P * m * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(w.ctr, 0, 24, s));
    k_source_caps<<<(P + 255) / 256, 256, 0, s>>>(cl.stage, rows, cols, m, lo, hi, *energy, w.ctr);
    const int lp = lanes_for(m);
    const long long nel = (long long)P * lp;
    k_to_colmajor<<<(unsigned)((nel + 255) / 256), 256, 0, s>>>(cl.stage, P, m, lp, w.vol);
    CK(cudaGetLastError());
    unsigned long long census[3];
    CK(cudaMemcpyAsync(census, w.ctr, 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaFree(cl.stage));
    cl.stage = nullptr;
    const unsigned long long lim = 0x7fffffffull;
    int hcap = HARD_CAP_DEFAULT;
    if (energy->hard_inhibit) {
        unsigned long long hc = 1ull << 16;
        while (hc <= census[0]) hc <<= 1;
        if (census[0] >= lim || (census[1] + 1) * hc + census[0] >= lim) return GZ_ERR_OVERFLOW;
        hcap = (int)hc;
    } else if (census[0] >= lim) {
        return GZ_ERR_OVERFLOW;
    }
    for (int k = 0; k < nbands; ++k) {
        CK(cudaSetDevice(devices[k]));
        CK(cudaStreamCreateWithFlags(&bp.stream[k], cudaStreamNonBlocking));
    }
    CK(cudaSetDevice(bp.home));
    unsigned long long h_ctr[gz::CTR_COUNT];
    Pending pd;
    rc = solve_launch(w, rows, cols, m, energy, sched, lo, hi, nullptr, s, hcap, 1, h_ctr, &pd,
                      lo ? (int)census[2] : -1, &bp);
    if (rc) return rc;
    CK(cudaMemcpyAsync(labels_host, w.labels, (size_t)P * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return solve_finish(pd, stats_out);
}

}  // extern "C"
