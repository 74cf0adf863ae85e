// odgs_b200_dropin.hpp — routes the reference's float hot path to the GPU, unchanged
// call sites included.
//
// Include AFTER the reference's headers (odgs/types.hpp, odgs/projection.hpp,
// odgs/rasterizer.hpp, odgs/backward.hpp). It declares non-template overloads for
// Scalar = float next to the reference's function templates in namespace odgs:
//
//   render, prepare_render          rasterizer.hpp:211-214, :129-132
//   backward                        backward.hpp:380-386
//   grad_pixels_to_splats           backward.hpp:208-211
//   project_gaussian                projection.hpp:178-181
//   cull                            rasterizer.hpp:15-18
//
// Overload resolution prefers a non-template exact match, so `odgs::render(cloud,
// camera, settings)` with float types — and the reference's own template callers such as
// train_step<float> (optimizer.hpp:107,112), found by argument-dependent lookup at
// instantiation — run on the GPU through the calling thread's context
// (odgs_b200::thread_context(), device $ODGS_B200_DEVICE). Double-precision calls keep
// the reference's CPU templates. Exceptions are the reference's.
#pragma once

#include "odgs_b200.hpp"

namespace odgs {

inline RenderOutput<float> render(const GaussianCloud<float>& cloud, const CameraPose<float>& camera,
                                  const RenderSettings<float>& settings) {
  return odgs_b200::render<RenderOutput<float>>(odgs_b200::thread_context(), cloud, camera, settings);
}

inline RenderOutput<float> prepare_render(const GaussianCloud<float>& cloud, const CameraPose<float>& camera,
                                          const RenderSettings<float>& settings) {
  return odgs_b200::prepare_render<RenderOutput<float>>(odgs_b200::thread_context(), cloud, camera, settings);
}

inline GradBuffers<float> backward(const GaussianCloud<float>& cloud, const CameraPose<float>& camera,
                                   const RenderOutput<float>& fwd, const ErpImage<float>& dl_dimage,
                                   const RenderSettings<float>& settings, const GradTSigns* signs = nullptr) {
  return odgs_b200::backward<GradBuffers<float>>(odgs_b200::thread_context(), cloud, camera, fwd, dl_dimage, settings,
                                                 signs);
}

inline std::vector<SplatGrads<float>> grad_pixels_to_splats(const RenderOutput<float>& fwd,
                                                            const ErpImage<float>& dl_dimage,
                                                            const RenderSettings<float>& settings) {
  return odgs_b200::grad_pixels_to_splats<SplatGrads<float>>(odgs_b200::thread_context(), fwd, dl_dimage, settings);
}

inline std::optional<Splat2D<float>> project_gaussian(const GaussianCloud<float>& cloud, Eigen::Index i,
                                                      const CameraPose<float>& camera,
                                                      const RenderSettings<float>& settings) {
  return odgs_b200::project_gaussian<Splat2D<float>>(odgs_b200::thread_context(), cloud, i, camera, settings);
}

inline std::vector<Eigen::Index> cull(const GaussianCloud<float>& cloud, const CameraPose<float>& camera,
                                      float near_radius, float far_radius) {
  return odgs_b200::cull<Eigen::Index>(odgs_b200::thread_context(), cloud, camera, near_radius, far_radius);
}

}  // namespace odgs
