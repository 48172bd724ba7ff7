// float64 instantiation (--fmad=false, like the physics and tail f64 units).
#include "go1env.cuh"
namespace dk { namespace go1 { DK_GO1_INSTANTIATE(double) } }
