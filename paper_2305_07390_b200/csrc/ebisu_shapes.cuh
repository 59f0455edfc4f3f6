// ebisu_shapes.cuh -- compile-time tap patterns, in the reference's catalog
// order (pkg/src/stencilplan/shapes.py:91-140).  The order fixes the
// summation order, which is what makes exact mode bitwise equal to the
// numpy oracle.  Specialised kernels are instantiated per shape; the host
// matcher (ebisu_api.cu) selects one only if the caller's tap list is
// identical, offset for offset, in the same order -- otherwise the generic
// runtime-tap kernel runs.
#pragma once

#include <utility>

namespace ebisu {

struct Off {
  int d0, d1, d2;  // axis 0 (streaming), axis 1, axis 2
};

// _star(dims, rad): axis-0 column -r..r first, then -r..-1,1..r per other axis
template <int DIMS, int RAD>
struct StarShape {
  static constexpr int dims = DIMS;
  static constexpr int R = RAD;
  static constexpr int NT = (2 * RAD + 1) + (DIMS - 1) * 2 * RAD;
  static constexpr bool kStar = true;
  __host__ __device__ static constexpr Off tap(int i) {
    if (i < 2 * R + 1) return Off{i - R, 0, 0};
    const int j = i - (2 * R + 1);
    const int axis = 1 + j / (2 * R);
    const int k = j % (2 * R);
    const int d = k < R ? k - R : k - R + 1;
    return axis == 1 ? Off{0, d, 0} : Off{0, 0, d};
  }
};

// _box(dims, rad): lexicographic product
template <int DIMS, int RAD>
struct BoxShape {
  static constexpr int dims = DIMS;
  static constexpr int R = RAD;
  static constexpr int W = 2 * RAD + 1;
  static constexpr int NT = DIMS == 1 ? W : (DIMS == 2 ? W * W : W * W * W);
  static constexpr bool kStar = false;
  __host__ __device__ static constexpr Off tap(int i) {
    if (DIMS == 1) return Off{i - R, 0, 0};
    if (DIMS == 2) return Off{i / W - R, i % W - R, 0};
    return Off{i / (W * W) - R, (i / W) % W - R, i % W - R};
  }
};

// _no_corners(3) (19 taps) and _j3d17pt (no corners, no +-axis-0 faces)
template <bool DropAxis0Faces>
struct NoCornerShape3 {
  static constexpr int dims = 3;
  static constexpr int R = 1;
  static constexpr int NT = DropAxis0Faces ? 17 : 19;
  static constexpr bool kStar = false;
  __host__ __device__ static constexpr bool keep(int a, int b, int c) {
    const int m = (a < 0 ? -a : a) + (b < 0 ? -b : b) + (c < 0 ? -c : c);
    if (m > 2) return false;
    if (DropAxis0Faces && b == 0 && c == 0 && a != 0) return false;
    return true;
  }
  __host__ __device__ static constexpr Off tap(int i) {
    int n = 0;
    for (int a = -1; a <= 1; ++a)
      for (int b = -1; b <= 1; ++b)
        for (int c = -1; c <= 1; ++c)
          if (keep(a, b, c)) {
            if (n == i) return Off{a, b, c};
            ++n;
          }
    return Off{0, 0, 0};
  }
};

// Shape ids shared with the host matcher.
enum ShapeId : int {
  SHAPE_J2D5PT = 0,    // StarShape<2,1>
  SHAPE_J2D9PT = 1,    // StarShape<2,2>
  SHAPE_J2D9PT_GOL = 2,  // BoxShape<2,1>
  SHAPE_J2D25PT = 3,   // BoxShape<2,2>
  SHAPE_J2D13PT = 4,   // StarShape<2,3>
  SHAPE_J2DS25PT = 5,  // StarShape<2,6>
  SHAPE_J3D7PT = 6,    // StarShape<3,1>
  SHAPE_J3D13PT = 7,   // StarShape<3,2>
  SHAPE_J3D17PT = 8,   // NoCornerShape3<true>
  SHAPE_J3D27PT = 9,   // BoxShape<3,1>
  SHAPE_POISSON = 10,  // NoCornerShape3<false>
  SHAPE_J1D3PT = 11,   // StarShape<1,1>
  SHAPE_COUNT = 12,
  SHAPE_GENERIC = -1
};

// compile-time loop: f(std::integral_constant<int, I>) for I in [0, N)
template <class F, int... Is>
__host__ __device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__host__ __device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

}  // namespace ebisu
