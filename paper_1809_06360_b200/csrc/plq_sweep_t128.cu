// K1 sweep kernel instantiated for 128-thread CTAs (body: plq_sweep_impl.cuh).
#include "plq_sweep_impl.cuh"

namespace plq {
PLQ_SWEEP_INSTANTIATE(128)
}  // namespace plq
