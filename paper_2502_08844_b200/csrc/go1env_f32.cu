// float32 instantiation of the fused Go1 joystick env step (go1env.cuh).
#include "go1env.cuh"
namespace dk { namespace go1 { DK_GO1_INSTANTIATE(float) } }
