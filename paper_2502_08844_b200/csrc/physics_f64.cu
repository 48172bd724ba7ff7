// float64 instantiation (built with --fmad=false: every a*b+c rounds twice,
// like the oracle's -ffp-contract=off, so forward kinematics and collision
// distances follow the oracle's arithmetic exactly).
#include "physics.cuh"
namespace dk { namespace phys { DK_PHYS_INSTANTIATE(double) } }
