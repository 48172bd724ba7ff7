// float64 instantiation of the env-step kernels.  Built with --fmad=false:
// every a*b+c rounds twice, as in the reference's Python float arithmetic.
#include "envstep_launch.cuh"
namespace dk {
DK_INSTANTIATE_LAUNCHERS(double)
}
