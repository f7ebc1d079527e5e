// Binding of the generic (runtime-shaped) decoder: used for every valid
// shape without a compile-time specialisation (rmfht_plan.h RMFHT_CHUNK*).
#include "rmfht_generic.cuh"
#include "rmfht_plan.h"

using rmfht_internal::fail;

namespace {

template <typename T>
rmfht_gen::Shape shape_of(const rmfht_plan* p) {
    return rmfht_gen::Shape{p->r, p->m, p->L, 1 << p->m, p->S};
}

template <typename T>
size_t smem_of(const rmfht_plan* p, int nw) {
    const auto lay = rmfht_gen::layout<T>(shape_of<T>(p));
    return (((size_t)(1 << p->m) * sizeof(T) + 15) / 16) * 16 + (size_t)lay.total * nw;
}

template <typename T>
int launch_gen(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm, int32_t* att,
               int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* /*work: none*/, cudaStream_t st) {
    rmfht::Params<T> prm;
    prm.llr = static_cast<const T*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = p->perms;
    prm.tie_fix = p->tie_fix;
    prm.cw = cw;
    prm.pm = static_cast<T*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<T*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    const auto sh = shape_of<T>(p);
    const auto lay = rmfht_gen::layout<T>(sh);
    const long long grid = B < p->grid ? B : p->grid;
    rmfht_gen::decode_kernel_generic<T><<<(unsigned)grid, p->nwarps * 32, p->smem, st>>>(prm, sh, lay);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("generic decode launch: ") + cudaGetErrorString(e));
    return 0;
}

template <typename T>
int prepare_gen(rmfht_plan* p) {
    const int Meff = p->perms ? p->M : 1;
    int nw = Meff < 4 ? Meff : 4;
    while (nw > 1 && smem_of<T>(p, nw) > 200 * 1024) nw--;
    const size_t smem = smem_of<T>(p, nw);
    auto kern = rmfht_gen::decode_kernel_generic<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "generic kernel does not fit an SM");
    p->nwarps = nw;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

}  // namespace

// Binds the generic kernel when the shape fits its limits; RMFHT_EUNSUPPORTED otherwise.
int rmfht_bind_generic(rmfht_plan* p) {
    if (p->m > 10 || p->L > rmfht_gen::kMaxL) return RMFHT_EUNSUPPORTED;
    const bool f64 = p->dtype == RMFHT_F64;
    const size_t need = f64 ? smem_of<double>(p, 1) : smem_of<float>(p, 1);
    if (need > 220 * 1024) return RMFHT_EUNSUPPORTED;
    p->fast = 0;
    p->generic = 1;
    if (f64) {
        p->launch = &launch_gen<double>;
        p->prepare = &prepare_gen<double>;
    } else {
        p->launch = &launch_gen<float>;
        p->prepare = &prepare_gen<float>;
    }
    return 0;
}
