// Store-pattern probe for the stage-(i) fill (diagnostics, not part of the
// product): how fast can 729-double rows be written with the access patterns
// k_build / k_expand use?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// scripts/store_probe.cu -o /tmp/store_probe && /tmp/store_probe
#include <cstdio>
#include <cuda_runtime.h>

// (a) warp per row, lane-strided 8-byte streaming stores (k_build's fill)
__global__ void rows8(double* out, long long nrows, int R) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (long long r = warp; r < nrows; r += nw) {
        double* o = out + r * R;
        for (int t = lane; t < R; t += 32) __stcs(o + t, 1.0 + t);
    }
}

// (a2) warp per row, lane pairs: 16-byte stores (rows 16-byte aligned: R even)
__global__ void rows16(double* out, long long nrows, int R) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (long long r = warp; r < nrows; r += nw) {
        double2* o = reinterpret_cast<double2*>(out + r * R);
        for (int t = lane; t < R / 2; t += 32) __stcs(o + t, make_double2(1.0 + t, 2.0 + t));
    }
}

// (b) same, default (write-back) stores
__global__ void rows8wb(double* out, long long nrows, int R) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (long long r = warp; r < nrows; r += nw) {
        double* o = out + r * R;
        for (int t = lane; t < R; t += 32) o[t] = 1.0 + t;
    }
}

// (c) flat grid-stride 16-byte stores over the whole buffer (the ceiling)
__global__ void flat16(double2* out, long long n2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
        __stcs(out + i, make_double2(1.0, 2.0));
}

// (d) flat grid-stride 8-byte stores
__global__ void flat8(double* out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        __stcs(out + i, 1.0);
}

// (e) CTA-contiguous: each CTA writes a contiguous range of rows, warp per row
__global__ void rows8c(double* out, long long nrows, int R, long long per_cta) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const long long r0 = blockIdx.x * per_cta;
    for (long long r = r0 + warp; r < r0 + per_cta && r < nrows; r += nw) {
        double* o = out + r * R;
        for (int t = lane; t < R; t += 32) __stcs(o + t, 1.0 + t);
    }
}

// (f) CTA per row-batch, the whole CTA writes rows contiguous chunk with lane-strided flat index
__global__ void batch_flat(double* out, long long nrows, int R, int rb) {
    for (long long b0 = (long long)blockIdx.x * rb; b0 < nrows; b0 += (long long)gridDim.x * rb) {
        const long long nb = (b0 + rb <= nrows ? rb : nrows - b0) * (long long)R;
        double* o = out + b0 * R;
        for (long long e = threadIdx.x; e < nb; e += blockDim.x) __stcs(o + e, 1.0);
    }
}

int main() {
    const int R = 729;
    const long long nrows = 18534825;
    const size_t bytes = (size_t)nrows * R * 8;
    double* buf;
    if (cudaMalloc(&buf, bytes + 4096) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int k = 0; k < 5; ++k) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-44s %8.2f ms  %7.1f GB/s  (%s)\n", name, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int per : {1, 2, 3}) {
        char nm[64];
        snprintf(nm, sizeof nm, "rows8 evict-first, %d CTAs/SM x256", per);
        run(nm, [&] { rows8<<<sms * per, 256>>>(buf, nrows, R); });
        snprintf(nm, sizeof nm, "rows16 (R=728) %d CTAs/SM x256", per);
        run(nm, [&] { rows16<<<sms * per, 256>>>(buf, nrows, 728); });
    }
    for (int per : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, sizeof nm, "rows8 evict-first, %d CTAs/SM x256", per);
        run(nm, [&] { rows8<<<sms * per, 256>>>(buf, nrows, R); });
    }
    run("rows8 write-back, 8 CTAs/SM", [&] { rows8wb<<<sms * 8, 256>>>(buf, nrows, R); });
    run("rows8 R=728 (16B-aligned rows)", [&] { rows8<<<sms * 8, 256>>>(buf, nrows, 728); });
    run("rows8 R=736 (64B-aligned rows)", [&] { rows8<<<sms * 8, 256>>>(buf, nrows * 729 / 736, 736); });
    {
        const long long per = (nrows + sms * 8 - 1) / (sms * 8);
        run("rows8 CTA-contiguous ranges", [&] { rows8c<<<sms * 8, 256>>>(buf, nrows, R, per); });
    }
    run("batch_flat rb=48 (CTA-flat over its rows)", [&] { batch_flat<<<sms * 4, 256>>>(buf, nrows, R, 48); });
    run("flat8", [&] { flat8<<<sms * 8, 256>>>(buf, (long long)(bytes / 8)); });
    run("flat16", [&] { flat16<<<sms * 8, 256>>>((double2*)buf, (long long)(bytes / 16)); });
    cudaFree(buf);
    return 0;
}
