// float32 instantiation of the locomotion step-tail kernels.
#include "locomotion.cuh"
namespace dk {
DK_LOCO_LAUNCHERS(, float)
}
