// K1 sweep kernel instantiated for 512-thread CTAs (body: plq_sweep_impl.cuh).
#include "plq_sweep_impl.cuh"

namespace plq {
PLQ_SWEEP_INSTANTIATE(512)
}  // namespace plq
