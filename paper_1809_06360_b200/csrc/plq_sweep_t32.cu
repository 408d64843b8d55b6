// K1 sweep kernel instantiated for 32-thread CTAs (body: plq_sweep_impl.cuh).
#include "plq_sweep_impl.cuh"

namespace plq {
PLQ_SWEEP_INSTANTIATE(32)
}  // namespace plq
