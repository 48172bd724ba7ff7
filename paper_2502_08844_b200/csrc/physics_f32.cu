// float32 instantiation of the articulated physics step (physics.cuh).
#include "physics.cuh"
namespace dk { namespace phys { DK_PHYS_INSTANTIATE(float) } }
