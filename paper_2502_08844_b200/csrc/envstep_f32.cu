// float32 instantiation of the env-step kernels (FMA contraction allowed).
#include "envstep_launch.cuh"
namespace dk {
DK_INSTANTIATE_LAUNCHERS(float)
}
