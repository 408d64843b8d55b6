// K1 sweep kernel instantiated for 256-thread CTAs (body: plq_sweep_impl.cuh).
#include "plq_sweep_impl.cuh"

namespace plq {
PLQ_SWEEP_INSTANTIATE(256)
}  // namespace plq
