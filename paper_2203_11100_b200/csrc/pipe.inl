// pipe.inl -- host side of the pipe-rate microbenchmark (swb_measure_pipe_rates).  Included by cabi.cu.

// ---- pipe-rate microbenchmark -------------------------------------------------------------------
template <int OP>
static swb_status run_pipe(int sm_count, double seconds, double* rate_ginst, double* clock_mhz) {
    uint32_t* sink = nullptr;
    unsigned long long* cyc = nullptr;
    SWB_CUDA(cudaMalloc(&sink, 64));
    SWB_CUDA(cudaMalloc(&cyc, sizeof(unsigned long long)));
    cudaEvent_t a, b;
    SWB_CUDA(cudaEventCreate(&a));
    SWB_CUDA(cudaEventCreate(&b));
    const int grid = sm_count * 2, block = 512;
    int iters = 2000;
    double ms = 0;
    for (int attempt = 0; attempt < 6; ++attempt) {
        SWB_CUDA(cudaMemset(cyc, 0, sizeof(unsigned long long)));
        pipe_rate_kernel<OP><<<grid, block>>>(sink, cyc, 0xfffefffeu, 0x00030003u, iters);   // warm-up
        SWB_CUDA(cudaMemset(cyc, 0, sizeof(unsigned long long)));
        SWB_CUDA(cudaEventRecord(a));
        pipe_rate_kernel<OP><<<grid, block>>>(sink, cyc, 0xfffefffeu, 0x00030003u, iters);
        SWB_CUDA(cudaEventRecord(b));
        SWB_CUDA(cudaEventSynchronize(b));
        float fms = 0;
        SWB_CUDA(cudaEventElapsedTime(&fms, a, b));
        ms = fms;
        if (ms >= seconds * 1000.0 * 0.5 || iters > (1 << 28)) break;
        const double scale = std::min(64.0, std::max(2.0, seconds * 1000.0 / std::max(ms, 1e-3)));
        iters = static_cast<int>(iters * scale);
    }
    unsigned long long cycles = 0;
    SWB_CUDA(cudaMemcpy(&cycles, cyc, sizeof(cycles), cudaMemcpyDeviceToHost));
    const double inst = static_cast<double>(grid) * block * static_cast<double>(iters) * kPipeChains * kPipeUnroll;
    *rate_ginst = inst / (ms * 1e-3) / 1e9;
    *clock_mhz = static_cast<double>(cycles) / (ms * 1e-3) / 1e6;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    cudaFree(cyc);
    return SWB_OK;
}

extern "C" {

swb_status swb_measure_pipe_rates(int32_t device, double seconds, swb_pipe_rates* out) {
    if (!out) return fail(SWB_ERR_INVALID, "out is null");
    std::memset(out, 0, sizeof(*out));
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SWB_ERR_CUDA, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(SWB_ERR_INVALID, "device index out of range");
    DeviceGuard guard(device);
    cudaDeviceProp prop{};
    SWB_CUDA(cudaGetDeviceProperties(&prop, device));
    out->sm_count = prop.multiProcessorCount;
    // half of the budget goes to the instruction the roofline is defined on, best of two runs (the first launch
    // after an idle period can still see the clock ramping); the rest is shared by the other probes
    const double each = std::max(0.02, seconds * 0.5 / (kOpCount - 1));
    double clk = 0, clk_sum = 0;
    swb_status st;
    for (int rep = 0; rep < 2; ++rep) {
        double rate = 0, c = 0;
        if ((st = run_pipe<kOpViaddmnmx16>(prop.multiProcessorCount, std::max(0.02, seconds * 0.25), &rate, &c)) != SWB_OK) return st;
        if (rate > out->viaddmnmx_s16x2) out->viaddmnmx_s16x2 = rate, clk_sum = c;
    }
    if ((st = run_pipe<kOpVimnmx3_16>(prop.multiProcessorCount, each, &out->vimnmx3_s16x2, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpViadd16>(prop.multiProcessorCount, each, &out->viadd_16x2, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpViaddmnmx32>(prop.multiProcessorCount, each, &out->viaddmnmx_s32, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpPrmt>(prop.multiProcessorCount, each, &out->prmt, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpImad>(prop.multiProcessorCount, each, &out->imad, &clk)) != SWB_OK) return st;
    if ((st = run_pipe<kOpMixAluFma>(prop.multiProcessorCount, each, &out->mix_alu_fma, &clk)) != SWB_OK) return st;
    out->sm_clock_mhz = clk_sum;
    return SWB_OK;
}

}  // extern "C"
