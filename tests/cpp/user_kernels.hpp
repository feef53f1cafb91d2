// User pair kernels (make_pair_kernel, pair_kernel.hpp:81-91) shared by the reference
// side (host, g++ against /root/reference/proj/include, namespace renamed) and the
// B200 drop-in side (nvcc; the pair functions are __host__ __device__ functors): a
// weighted sum over an input field, min / max reductions, and a postamble.
#pragma once
#include <array>
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define SFCNL_HD __host__ __device__
#else
#define SFCNL_HD
#endif

template <class Real>
struct UkWeighted {  // sum_j m_j (1 - d2 / h_i^2), sum_j m_i dx / h_i
    SFCNL_HD std::array<Real, 2> operator()(const sfcnl::PairArgs<Real>& a, const std::array<Real, 1>& in_i,
                                            const std::array<Real, 1>& in_j) const {
        const Real q2 = a.d2 / (a.h_i * a.h_i);
        return std::array<Real, 2>{in_j[0] * (Real(1) - q2), in_i[0] * a.dx.x / a.h_i};
    }
};

template <class Real>
struct UkMinMax {  // nearest distance, largest dz
    SFCNL_HD std::array<Real, 2> operator()(const sfcnl::PairArgs<Real>& a, const std::array<Real, 0>&,
                                            const std::array<Real, 0>&) const {
        return std::array<Real, 2>{std::sqrt(a.d2), a.dx.z};
    }
};

template <class Real>
struct UkHj {
    SFCNL_HD std::array<Real, 1> operator()(const sfcnl::PairArgs<Real>& a, const std::array<Real, 0>&,
                                            const std::array<Real, 0>&) const {
        return std::array<Real, 1>{a.h_j};
    }
};
template <class Real>
struct UkMean {  // postamble: mean h_j over the neighbourhood
    SFCNL_HD void operator()(std::size_t i, std::array<Real, 1>& v, std::uint32_t count) const {
        v[0] = count ? v[0] / Real(count) : Real(i % 7);
    }
};

template <class Real>
auto uk_weighted() {
    return sfcnl::make_pair_kernel<Real, 1, 2>(
        {"m"}, {sfcnl::OutputSpec{"w", sfcnl::Symmetry::even, sfcnl::Reduction::sum},
                sfcnl::OutputSpec{"gx", sfcnl::Symmetry::odd, sfcnl::Reduction::sum}},
        UkWeighted<Real>{});
}

template <class Real>
auto uk_minmax() {
    return sfcnl::make_pair_kernel<Real, 0, 2>(
        {}, {sfcnl::OutputSpec{"dmin", sfcnl::Symmetry::even, sfcnl::Reduction::min},
             sfcnl::OutputSpec{"dzmax", sfcnl::Symmetry::odd, sfcnl::Reduction::max}},
        UkMinMax<Real>{});
}

template <class Real>
auto uk_post() {
    return sfcnl::make_pair_kernel<Real, 0, 1>(
        {}, {sfcnl::OutputSpec{"hmean", sfcnl::Symmetry::even, sfcnl::Reduction::sum}}, UkHj<Real>{}, UkMean<Real>{});
}
