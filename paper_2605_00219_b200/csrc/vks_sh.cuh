// vks_sh.cuh — the real spherical-harmonics basis constants of degrees 0-3 (3DGS convention:
// Y_0 = C0, Y_1..3 = -C1 y, C1 z, -C1 x, ...; DESIGN.md §4.1 step 12), shared by the projection
// forward (project.cu) and backward (project_bwd.cu).  Closed-form values, rounded to fp32.
#pragma once

namespace vks {
namespace sh {
constexpr float C0 = 0.28209479177387814f;
constexpr float C1 = 0.4886025119029199f;
constexpr float C20 = 1.0925484305920792f;
constexpr float C21 = -1.0925484305920792f;
constexpr float C22 = 0.31539156525252005f;
constexpr float C23 = -1.0925484305920792f;
constexpr float C24 = 0.5462742152960396f;
constexpr float C30 = -0.5900435899266435f;
constexpr float C31 = 2.890611442640554f;
constexpr float C32 = -0.4570457994644658f;
constexpr float C33 = 0.3731763325901154f;
constexpr float C34 = -0.4570457994644658f;
constexpr float C35 = 1.445305721320277f;
constexpr float C36 = -0.5900435899266435f;
}  // namespace sh
}  // namespace vks
