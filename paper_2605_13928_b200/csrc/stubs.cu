// Entry points not implemented yet in this build (return SCB_ERR_UNSUPPORTED).
#include "common.cuh"
#define STUB(name, ...) extern "C" int name(__VA_ARGS__) { scb::set_error(#name ": not implemented"); return SCB_ERR_UNSUPPORTED; }




STUB(scb_synth_rows, scb_ctx*, uint64_t, int64_t, int64_t, int32_t, const double*, const double*, int32_t, const double*, int32_t, const double*, const int64_t*, int64_t*, int32_t*, float*, void*)
