// K2+K3 instantiations for model kind 1 (see k23_launch.cuh).
#include "k23_launch.cuh"
namespace d4k {
D4K_INSTANTIATE_K23(1)
}
