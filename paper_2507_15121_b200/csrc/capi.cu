#include <algorithm>
// capi.cu -- error plumbing and device queries for the C ABI.
#include <stdarg.h>

#include "common.cuh"

#include <cxxabi.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace skrp {

static thread_local char g_err[512] = {0};
static thread_local int g_err_code = 0;

void set_error(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    g_err_code = code;
}

int cuda_status(cudaError_t e, const char *where)
{
    int code = (e == cudaErrorMemoryAllocation) ? SKRP_ERR_NOMEM : SKRP_ERR_CUDA;
    set_error(code, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
    return code;
}

int device_sm_count()
{
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return sms;
}

namespace {
std::mutex g_log_mu;
std::vector<std::string> g_log;
constexpr size_t kLogMax = 4096;
}  // namespace

void note_launch(const void *kernel, int mode)
{
    const char *mangled = nullptr;
    std::string name = "?";
    if (cudaFuncGetName(&mangled, kernel) == cudaSuccess && mangled) {
        int st = 0;
        char *dm = abi::__cxa_demangle(mangled, nullptr, nullptr, &st);
        name = (st == 0 && dm) ? dm : mangled;
        free(dm);
    }
    std::lock_guard<std::mutex> lk(g_log_mu);
    if (g_log.size() < kLogMax) g_log.push_back(std::to_string(mode) + "\t" + name);
}

}  // namespace skrp

extern "C" {

int skrp_launch_log(int64_t index, char *buf, size_t len, int64_t *count)
{
    std::lock_guard<std::mutex> lk(skrp::g_log_mu);
    if (count) *count = (int64_t)skrp::g_log.size();
    if (index < 0) {  // clear
        skrp::g_log.clear();
        return SKRP_OK;
    }
    SKRP_REQUIRE(index < (int64_t)skrp::g_log.size(), "launch log has %zu entries, asked for %lld",
                 skrp::g_log.size(), (long long)index);
    SKRP_REQUIRE(buf != nullptr && len > 0, "skrp_launch_log: null buffer");
    snprintf(buf, len, "%s", skrp::g_log[(size_t)index].c_str());
    return SKRP_OK;
}

int skrp_last_error(char *buf, size_t len)
{
    if (buf && len) {
        strncpy(buf, skrp::g_err, len - 1);
        buf[len - 1] = 0;
    }
    return skrp::g_err_code;
}

int skrp_abi_version(void) { return 12; }

int skrp_device_sm_count(int *out)
{
    SKRP_REQUIRE(out != nullptr, "skrp_device_sm_count: null output");
    int dev = 0;
    SKRP_CUDA(cudaGetDevice(&dev));
    SKRP_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
    return SKRP_OK;
}

// ------------------------------------------------------------- CUDA IPC
// Peer output buffers for the fused all-gather push: a torch allocation is a
// slice of a larger cudaMalloc segment, so the handle is taken on the
// segment base (cuMemGetAddressRange through the runtime's driver entry
// point -- no -lcuda) and the slice offset travels with it.
typedef int (*MemGetAddressRangeFn)(unsigned long long *, size_t *, unsigned long long);

int skrp_ipc_get_handle(const void *dev_ptr, uint8_t *handle64, int64_t *offset)
{
    SKRP_REQUIRE(dev_ptr && handle64 && offset, "skrp_ipc_get_handle: null pointer");
    static MemGetAddressRangeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        SKRP_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
        SKRP_REQUIRE(f && q == cudaDriverEntryPointSuccess, "cuMemGetAddressRange unavailable");
        fn = (MemGetAddressRangeFn)f;
    }
    unsigned long long base = 0;
    size_t size = 0;
    SKRP_REQUIRE(fn(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) == 0, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    SKRP_CUDA(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
    memcpy(handle64, &h, sizeof(h));
    *offset = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return SKRP_OK;
}

int skrp_ipc_open_handle(const uint8_t *handle64, int64_t offset, void **dev_ptr, void **base_out)
{
    SKRP_REQUIRE(handle64 && dev_ptr && base_out && offset >= 0, "skrp_ipc_open_handle: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    void *base = nullptr;
    SKRP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *base_out = base;
    *dev_ptr = (void *)((uintptr_t)base + (uintptr_t)offset);
    return SKRP_OK;
}

int skrp_ipc_close_handle(void *base)
{
    SKRP_REQUIRE(base != nullptr, "skrp_ipc_close_handle: null pointer");
    SKRP_CUDA(cudaIpcCloseMemHandle(base));
    return SKRP_OK;
}

}  // extern "C"
