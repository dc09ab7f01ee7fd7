// svn_eigen_subset.hpp — TEST INFRASTRUCTURE ONLY (oracle/ref, the reference build recipe).
//
// A small, independently written implementation of the part of the Eigen 3 API that the
// reference's own sources use (/root/reference/proj: include/sweptnet/*.hpp, src/nn.cpp,
// src/robot.cpp, src/geometry.cpp).  Eigen3 is absent from this image and from the GPU boxes
// (SURVEY.md §8c), so without it the reference's inference code cannot be compiled; with this
// header it compiles UNMODIFIED and is run here as the parity oracle's own oracle.
//
// Evaluation model.  Like Eigen, coefficient-wise expressions are lazy: an assignment
// `dst op= expr` runs one loop whose body is the whole expression for one coefficient, so
// GCC's -ffp-contract=fast (the reference builds -std=gnu++20 -O3 -march=native,
// CMakeLists.txt:3,31-38) fuses a multiply feeding an add into one FMA exactly where it would
// in Eigen's evaluators (e.g. nn.cpp:119,123-124 `a += h[k] * W.col(k)` -> fma(h_k, W_ik, a_i);
// nn.cpp:125 -> h + fma(max(a,0), s, t); nn.cpp:110 beta - mean*scale -> fma(-mean, scale, beta)).
// Element-wise results do not depend on SIMD width, so they match Eigen's vectorised paths.
// Reductions are where vectorisation changes the ORDER: Eigen's scalar (non-vectorised)
// redux is sequential, `res = c0; res = res + c_k` (k ascending) — implemented here as the
// default, every term rounded before it is added (see redux()).  With SVN_EIGEN_PACKET_REDUX=W (W = 4, 8 or 16 lanes) `dot`/`sum` instead follow
// the structure of Eigen's linear-vectorised redux (two W-lane partial sums over the aligned
// body, combined, then a horizontal tree and the scalar tail) so the ulp effect of the
// ISA-dependent order at nn.cpp:127 can be measured (tests/test_ref_oracle.py).
// Matrix products (training path only) are evaluated eagerly, k ascending.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

#ifndef SVN_EIGEN_PACKET_REDUX
#define SVN_EIGEN_PACKET_REDUX 0
#endif

#define SVN_EI inline __attribute__((always_inline))
#define SVN_EIL __attribute__((always_inline))

namespace Eigen {

using Index = std::ptrdiff_t;
inline constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };
enum NoChange_t { NoChange };

template <class D> struct DenseBase;
template <class S, int R, int C, int Opt, int MR, int MC> class Matrix;

namespace internal {
template <class T> struct is_plain : std::false_type {};
template <class S, int R, int C, int O, int MR, int MC> struct is_plain<Matrix<S, R, C, O, MR, MC>> : std::true_type {};
// leaves (plain matrices) are held by reference, expressions by value (as in Eigen)
template <class T> using nested = std::conditional_t<is_plain<std::remove_cv_t<T>>::value, const T&, T>;
template <class T> concept Expr = std::is_base_of_v<DenseBase<std::remove_cvref_t<T>>, std::remove_cvref_t<T>>;
template <int R, int C> constexpr int default_opts() { return (R == 1 && C != 1) ? RowMajor : ColMajor; }

// Coefficient storage.  Fixed sizes are stored inline with no other members, like Eigen's
// (sizeof(Vector3d) == 24, so a std::vector<Vector3d> is a contiguous double [n x 3] — the
// layout the reference's callers hand to the C-ABI); dynamic sizes on the heap.
template <class S, int R, int C, bool Fixed = (R > 0 && C > 0)>
struct DenseStorage {
    std::array<S, static_cast<size_t>(R > 0 && C > 0 ? R * C : 1)> d{};
    static constexpr Index rows() { return R; }
    static constexpr Index cols() { return C; }
    S* data() { return d.data(); }
    const S* data() const { return d.data(); }
    void set(Index r, Index c) {
        if (r != R || c != C) throw std::invalid_argument("svn eigen subset: resizing a fixed-size matrix");
        d.fill(S(0));
    }
    void swap(DenseStorage& o) noexcept { d.swap(o.d); }
};
template <class S, int R, int C>
struct DenseStorage<S, R, C, false> {
    Index r = R > 0 ? R : 0, c = C > 0 ? C : 0;  // declared before d: initialised first
    std::vector<S> d;
    DenseStorage() : d(static_cast<size_t>(r * c)) {}
    Index rows() const { return r; }
    Index cols() const { return c; }
    S* data() { return d.data(); }
    const S* data() const { return d.data(); }
    void set(Index rr, Index cc) {
        if ((R > 0 && rr != R) || (C > 0 && cc != C)) throw std::invalid_argument("svn eigen subset: resizing a fixed dimension");
        r = rr;
        c = cc;
        d.assign(static_cast<size_t>(rr * cc), S(0));
    }
    void swap(DenseStorage& o) noexcept {
        d.swap(o.d);
        std::swap(r, o.r);
        std::swap(c, o.c);
    }
};
}  // namespace internal

// ------------------------------------------------------------------------------------------
// Reductions: sequential (Eigen's scalar redux) or packet-structured (see header comment).
namespace internal {
template <class S, class F>
SVN_EI S redux(Index n, F&& coeff) {
#if SVN_EIGEN_PACKET_REDUX > 0
    constexpr Index W = SVN_EIGEN_PACKET_REDUX;
    if (std::is_same_v<S, float> && n >= W) {
        const Index body2 = (n / (2 * W)) * (2 * W), body = (n / W) * W;
        S p0[W], p1[W];
        for (Index l = 0; l < W; ++l) p0[l] = coeff(l);
        if (body > W) {
            for (Index l = 0; l < W; ++l) p1[l] = coeff(W + l);
            for (Index i = 2 * W; i < body2; i += 2 * W)
                for (Index l = 0; l < W; ++l) {
                    p0[l] = p0[l] + coeff(i + l);
                    p1[l] = p1[l] + coeff(i + W + l);
                }
            for (Index l = 0; l < W; ++l) p0[l] = p0[l] + p1[l];
            if (body > body2)
                for (Index l = 0; l < W; ++l) p0[l] = p0[l] + coeff(body2 + l);
        }
        // horizontal: fold halves (lane l + lane l+w/2) down to one lane
        for (Index w = W; w > 1; w /= 2)
            for (Index l = 0; l < w / 2; ++l) p0[l] = p0[l] + p0[l + w / 2];
        S res = p0[0];
        for (Index i = body; i < n; ++i) res = res + coeff(i);
        return res;
    }
#endif
    // Each term is rounded on its own, then added in index order: what g++ -O3 makes of
    // Eigen's scalar redux when it vectorises the in-order reduction (the product is a
    // vector multiply, the adds stay sequential, nothing is fused).  The volatile makes that
    // explicit, so the result does not hinge on the vectoriser's cost model for a given type.
    S res = coeff(0);
    for (Index i = 1; i < n; ++i) {
        volatile S term = coeff(i);
        res = res + term;
    }
    return res;
}
}  // namespace internal

// ------------------------------------------------------------------------------------------
// Expression nodes
template <class F, class X> struct CwiseUnaryOp;
template <class F, class L, class R> struct CwiseBinaryOp;
template <class X> struct Transpose;
template <class X, bool A> struct KindView;
template <class X> struct Block;
template <class X> struct RowwiseOp;
template <class X> struct ColwiseOp;
template <class X> struct RowBroadcast;

namespace internal {
template <class L, class R> constexpr void check_same_kind() {
    static_assert(L::is_array == R::is_array, "svn eigen subset: mixing array and matrix expressions");
}
struct op_sum { template <class A, class B> SVN_EI auto operator()(A a, B b) const { return a + b; } };
struct op_diff { template <class A, class B> SVN_EI auto operator()(A a, B b) const { return a - b; } };
struct op_prod { template <class A, class B> SVN_EI auto operator()(A a, B b) const { return a * b; } };
struct op_quot { template <class A, class B> SVN_EI auto operator()(A a, B b) const { return a / b; } };
struct op_max { template <class A> SVN_EI A operator()(A a, A b) const { return std::max(a, b); } };
struct op_min { template <class A> SVN_EI A operator()(A a, A b) const { return std::min(a, b); } };
struct op_ge { template <class A> SVN_EI bool operator()(A a, A b) const { return a >= b; } };
struct op_le { template <class A> SVN_EI bool operator()(A a, A b) const { return a <= b; } };
struct op_gt { template <class A> SVN_EI bool operator()(A a, A b) const { return a > b; } };
struct op_lt { template <class A> SVN_EI bool operator()(A a, A b) const { return a < b; } };
template <class S> struct op_scal_r { S s; template <class A> SVN_EI auto operator()(A a) const { return a * s; } };
template <class S> struct op_scal_l { S s; template <class A> SVN_EI auto operator()(A a) const { return s * a; } };
template <class S> struct op_div_s { S s; template <class A> SVN_EI auto operator()(A a) const { return a / s; } };
template <class S> struct op_add_s { S s; template <class A> SVN_EI auto operator()(A a) const { return a + s; } };
template <class S> struct op_sub_s { S s; template <class A> SVN_EI auto operator()(A a) const { return a - s; } };
template <class S> struct op_max_s { S s; template <class A> SVN_EI A operator()(A a) const { return std::max(a, s); } };
template <class S> struct op_min_s { S s; template <class A> SVN_EI A operator()(A a) const { return std::min(a, s); } };
template <class S> struct op_cmp_gt_s { S s; template <class A> SVN_EI bool operator()(A a) const { return a > s; } };
template <class S> struct op_cmp_lt_s { S s; template <class A> SVN_EI bool operator()(A a) const { return a < s; } };
template <class S> struct op_cmp_ge_s { S s; template <class A> SVN_EI bool operator()(A a) const { return a >= s; } };
template <class S> struct op_cmp_le_s { S s; template <class A> SVN_EI bool operator()(A a) const { return a <= s; } };
struct op_neg { template <class A> SVN_EI A operator()(A a) const { return -a; } };
struct op_abs { template <class A> SVN_EI A operator()(A a) const { return std::abs(a); } };
struct op_abs2 { template <class A> SVN_EI A operator()(A a) const { return a * a; } };
struct op_sqrt { template <class A> SVN_EI A operator()(A a) const { return std::sqrt(a); } };
struct op_rsqrt { template <class A> SVN_EI A operator()(A a) const { return A(1) / std::sqrt(a); } };
template <class T> struct op_cast { template <class A> SVN_EI T operator()(A a) const { return static_cast<T>(a); } };
}  // namespace internal

// The common base of every expression: read access + the expression-building API.
template <class D>
struct DenseBase {
    SVN_EI const D& derived() const { return static_cast<const D&>(*this); }
    SVN_EI D& derived() { return static_cast<D&>(*this); }
    SVN_EI Index size() const { return derived().rows() * derived().cols(); }
    // linear access, vectors only (row or column)
    SVN_EI auto vcoeff(Index k) const { return derived().cols() == 1 ? derived().coeff(k, 0) : derived().coeff(0, k); }
    SVN_EI auto operator()(Index i, Index j) const { return derived().coeff(i, j); }
    SVN_EI auto operator[](Index k) const { return vcoeff(k); }
    SVN_EI auto x() const { return vcoeff(0); }
    SVN_EI auto y() const { return vcoeff(1); }
    SVN_EI auto z() const { return vcoeff(2); }

    // ---- views
    auto array() const { return KindView<internal::nested<D>, true>(derived()); }
    auto matrix() const { return KindView<internal::nested<D>, false>(derived()); }
    auto transpose() const { return Transpose<internal::nested<D>>(derived()); }
    auto row(Index i) const { return Block<const D>(&derived(), i, 0, 1, derived().cols()); }
    auto col(Index j) const { return Block<const D>(&derived(), 0, j, derived().rows(), 1); }
    auto leftCols(Index n) const { return Block<const D>(&derived(), 0, 0, derived().rows(), n); }
    auto rightCols(Index n) const { return Block<const D>(&derived(), 0, derived().cols() - n, derived().rows(), n); }
    auto head(Index n) const { return derived().cols() == 1 ? Block<const D>(&derived(), 0, 0, n, 1) : Block<const D>(&derived(), 0, 0, 1, n); }
    auto rowwise() const { return RowwiseOp<internal::nested<D>>(derived()); }
    auto colwise() const { return ColwiseOp<internal::nested<D>>(derived()); }

    // ---- coefficient-wise
    template <class O> auto cwiseProduct(const DenseBase<O>& o) const {
        return CwiseBinaryOp<internal::op_prod, internal::nested<D>, internal::nested<O>>(derived(), o.derived());
    }
    template <class O> auto cwiseQuotient(const DenseBase<O>& o) const {
        return CwiseBinaryOp<internal::op_quot, internal::nested<D>, internal::nested<O>>(derived(), o.derived());
    }
    template <class O> auto cwiseMax(const DenseBase<O>& o) const {
        return CwiseBinaryOp<internal::op_max, internal::nested<D>, internal::nested<O>>(derived(), o.derived());
    }
    template <class O> auto cwiseMin(const DenseBase<O>& o) const {
        return CwiseBinaryOp<internal::op_min, internal::nested<D>, internal::nested<O>>(derived(), o.derived());
    }
    template <class S> auto cwiseMax(S s) const { return unary(internal::op_max_s<typename D::Scalar>{typename D::Scalar(s)}); }
    template <class S> auto cwiseMin(S s) const { return unary(internal::op_min_s<typename D::Scalar>{typename D::Scalar(s)}); }
    auto cwiseAbs() const { return unary(internal::op_abs{}); }
    auto cwiseAbs2() const { return unary(internal::op_abs2{}); }
    auto abs() const { return unary(internal::op_abs{}); }
    auto square() const { return unary(internal::op_abs2{}); }
    auto sqrt() const { return unary(internal::op_sqrt{}); }
    auto rsqrt() const { return unary(internal::op_rsqrt{}); }
    template <class F> auto unaryExpr(F f) const { return unary(f); }
    template <class T> auto cast() const { return unary(internal::op_cast<T>{}); }
    template <class F> auto unary(F f) const { return CwiseUnaryOp<F, internal::nested<D>>(derived(), f); }

    // ---- reductions
    auto sum() const {
        using S = typename D::Scalar;
        const D& d = derived();
        if (d.rows() == 1 || d.cols() == 1) return internal::redux<S>(size(), [&](Index k) SVN_EIL { return d.vcoeff(k); });
        const Index r = d.rows();
        return internal::redux<S>(size(), [&](Index k) SVN_EIL { return d.coeff(k % r, k / r); });
    }
    auto mean() const { return sum() / static_cast<typename D::Scalar>(size()); }
    auto prod() const {
        const D& d = derived();
        typename D::Scalar res = d.coeff(0, 0);
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i)
                if (i || j) res = res * d.coeff(i, j);
        return res;
    }
    auto maxCoeff() const {
        const D& d = derived();
        typename D::Scalar res = d.coeff(0, 0);
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i) res = std::max(res, d.coeff(i, j));
        return res;
    }
    auto minCoeff() const {
        const D& d = derived();
        typename D::Scalar res = d.coeff(0, 0);
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i) res = std::min(res, d.coeff(i, j));
        return res;
    }
    bool all() const {
        const D& d = derived();
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i)
                if (!d.coeff(i, j)) return false;
        return true;
    }
    bool any() const {
        const D& d = derived();
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i)
                if (d.coeff(i, j)) return true;
        return false;
    }
    bool allFinite() const {
        const D& d = derived();
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i)
                if (!std::isfinite(d.coeff(i, j))) return false;
        return true;
    }
    template <class O> auto dot(const DenseBase<O>& o) const {
        using S = typename D::Scalar;
        const D& a = derived();
        const O& b = o.derived();
        if (a.size() != b.size()) throw std::invalid_argument("svn eigen subset: dot size mismatch");
        return internal::redux<S>(a.size(), [&](Index k) SVN_EIL { return a.vcoeff(k) * b.vcoeff(k); });
    }
    auto squaredNorm() const { return cwiseAbs2().sum(); }
    auto norm() const { return std::sqrt(squaredNorm()); }
    auto normalized() const { return unary(internal::op_div_s<typename D::Scalar>{norm()}); }
    auto eval() const { return Matrix<typename D::Scalar, Dynamic, Dynamic, ColMajor, Dynamic, Dynamic>(derived()); }

    // 3-vectors (geometry.cpp)
    template <class O> auto cross(const DenseBase<O>& o) const;
    auto unitOrthogonal() const;
    auto determinant() const {
        const D& m = derived();
        return m.coeff(0, 0) * (m.coeff(1, 1) * m.coeff(2, 2) - m.coeff(1, 2) * m.coeff(2, 1)) -
               m.coeff(0, 1) * (m.coeff(1, 0) * m.coeff(2, 2) - m.coeff(1, 2) * m.coeff(2, 0)) +
               m.coeff(0, 2) * (m.coeff(1, 0) * m.coeff(2, 1) - m.coeff(1, 1) * m.coeff(2, 0));
    }
};

// Writable expressions (plain matrices, blocks of them, array views of them): coefficient-wise
// assignment loops.  One loop per assignment, the whole right-hand side inlined per coefficient.
template <class D>
struct WritableBase : DenseBase<D> {
    using DenseBase<D>::derived;
    template <class E, class Op>
    SVN_EI void assign_loop(const E& e, Op op) {
        D& d = derived();
        const Index R = d.rows(), Cc = d.cols();
        if (e.rows() != R || e.cols() != Cc) throw std::invalid_argument("svn eigen subset: size mismatch in assignment");
        if constexpr (D::row_major) {
            for (Index i = 0; i < R; ++i)
                for (Index j = 0; j < Cc; ++j) op(d.coeffRef(i, j), e.coeff(i, j));
        } else {
            for (Index j = 0; j < Cc; ++j)
                for (Index i = 0; i < R; ++i) op(d.coeffRef(i, j), e.coeff(i, j));
        }
    }
    template <class E> D& operator+=(const DenseBase<E>& e) {
        assign_loop(e.derived(), [](auto& a, auto b) SVN_EIL { a = a + b; });
        return derived();
    }
    template <class E> D& operator-=(const DenseBase<E>& e) {
        assign_loop(e.derived(), [](auto& a, auto b) SVN_EIL { a = a - b; });
        return derived();
    }
    template <class E> D& operator*=(const DenseBase<E>& e) requires D::is_array {
        assign_loop(e.derived(), [](auto& a, auto b) SVN_EIL { a = a * b; });
        return derived();
    }
    template <class S> D& operator*=(S s) requires std::is_arithmetic_v<S> {
        for_each([&](auto& a) SVN_EIL { a = a * s; });
        return derived();
    }
    template <class S> D& operator/=(S s) requires std::is_arithmetic_v<S> {
        for_each([&](auto& a) SVN_EIL { a = a / s; });
        return derived();
    }
    template <class S> D& operator+=(S s) requires(std::is_arithmetic_v<S> && D::is_array) {
        for_each([&](auto& a) SVN_EIL { a = a + s; });
        return derived();
    }
    template <class S> D& operator-=(S s) requires(std::is_arithmetic_v<S> && D::is_array) {
        for_each([&](auto& a) SVN_EIL { a = a - s; });
        return derived();
    }
    template <class F> SVN_EI void for_each(F f) {
        D& d = derived();
        for (Index j = 0; j < d.cols(); ++j)
            for (Index i = 0; i < d.rows(); ++i) f(d.coeffRef(i, j));
    }
    SVN_EI auto& operator()(Index i, Index j) { return derived().coeffRef(i, j); }
    SVN_EI auto operator()(Index i, Index j) const { return derived().coeff(i, j); }
    SVN_EI auto& operator[](Index k) { return derived().cols() == 1 ? derived().coeffRef(k, 0) : derived().coeffRef(0, k); }
    SVN_EI auto operator[](Index k) const { return this->vcoeff(k); }
    SVN_EI auto& x() { return (*this)[0]; }
    SVN_EI auto& y() { return (*this)[1]; }
    SVN_EI auto& z() { return (*this)[2]; }
    SVN_EI auto x() const { return this->vcoeff(0); }
    SVN_EI auto y() const { return this->vcoeff(1); }
    SVN_EI auto z() const { return this->vcoeff(2); }
    void setZero() { for_each([](auto& a) { a = 0; }); }
    void setOnes() { for_each([](auto& a) { a = 1; }); }
};

// ------------------------------------------------------------------------------------------
// Matrix (dense, heap storage; fixed sizes are sized at construction)
template <class S, int R, int C, int Opt = internal::default_opts<R, C>(), int MR = R, int MC = C>
class Matrix : public WritableBase<Matrix<S, R, C, Opt, MR, MC>> {
public:
    using Scalar = S;
    static constexpr bool is_array = false;
    static constexpr bool row_major = (Opt & RowMajor) != 0;
    static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C;
    using Base = WritableBase<Matrix>;
    using Base::operator+=;
    using Base::operator-=;
    using Base::operator();
    using Base::operator[];
    using Base::x;
    using Base::y;
    using Base::z;
    using Base::setZero;
    using Base::setOnes;

    Matrix() = default;
    // dynamic: (rows, cols); vectors: (size)
    Matrix(Index rows, Index cols) requires(R == Dynamic || C == Dynamic) { resize(rows, cols); }
    explicit Matrix(Index n) requires((R == 1 || C == 1) && (R == Dynamic || C == Dynamic)) { resize(n); }
    // fixed 3-vectors
    Matrix(S a, S b, S c) requires(R * C == 3) {
        st_.d[0] = a;
        st_.d[1] = b;
        st_.d[2] = c;
    }
    template <class T0, class T1, class T2>
    Matrix(T0 a, T1 b, T2 c) requires(R * C == 3 && std::is_arithmetic_v<T0> && !std::is_same_v<T0, S>)
        : Matrix(S(a), S(b), S(c)) {}
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;
    template <class E> Matrix(const DenseBase<E>& e) { *this = e; }
    template <class E> Matrix& operator=(const DenseBase<E>& e) {
        const E& x = e.derived();
        Matrix tmp;
        tmp.resize(x.rows(), x.cols());
        tmp.assign_loop(x, [](auto& a, auto b) SVN_EIL { a = b; });
        st_.swap(tmp.st_);
        return *this;
    }

    SVN_EI Index rows() const { return st_.rows(); }
    SVN_EI Index cols() const { return st_.cols(); }
    SVN_EI Index idx(Index i, Index j) const { return row_major ? i * cols() + j : j * rows() + i; }
    SVN_EI S coeff(Index i, Index j) const { return st_.data()[idx(i, j)]; }
    SVN_EI S& coeffRef(Index i, Index j) { return st_.data()[idx(i, j)]; }
    SVN_EI S& operator[](Index k) { return st_.data()[k]; }
    SVN_EI S operator[](Index k) const { return st_.data()[k]; }
    SVN_EI S& operator()(Index k) { return st_.data()[k]; }
    SVN_EI S operator()(Index k) const { return st_.data()[k]; }
    S* data() { return st_.data(); }
    const S* data() const { return st_.data(); }

    void resize(Index rows, Index cols) { st_.set(rows, cols); }
    void resize(Index n) {
        static_assert(R == 1 || C == 1, "resize(n) on a matrix");
        if constexpr (C == 1) resize(n, 1); else resize(1, n);
    }
    void conservativeResize(Index rows, NoChange_t) { conservativeResize(rows, cols()); }
    void conservativeResize(Index n) {
        if constexpr (C == 1) conservativeResize(n, 1); else conservativeResize(1, n);
    }
    void conservativeResize(Index rows, Index cols) {
        Matrix m;
        m.resize(rows, cols);
        for (Index i = 0; i < std::min(rows, this->rows()); ++i)
            for (Index j = 0; j < std::min(cols, this->cols()); ++j) m.coeffRef(i, j) = coeff(i, j);
        st_.swap(m.st_);
    }
    void setZero(Index n) { resize(n), setZero(); }
    void setOnes(Index n) { resize(n), setOnes(); }
    void setZero(Index rows, Index cols) { resize(rows, cols), setZero(); }
    void swap(Matrix& o) noexcept { st_.swap(o.st_); }
    auto noalias() { return NoAlias{*this}; }
    struct NoAlias {
        Matrix& m;
        template <class E> Matrix& operator=(const DenseBase<E>& e) { return m = e; }
        template <class E> Matrix& operator+=(const DenseBase<E>& e) { return m += e; }
        template <class E> Matrix& operator-=(const DenseBase<E>& e) { return m -= e; }
    };

    // writable views of an lvalue matrix
    auto array() { return KindView<Matrix&, true>(*this); }
    auto array() const { return KindView<const Matrix&, true>(*this); }
    auto matrix() { return KindView<Matrix&, false>(*this); }
    auto matrix() const { return KindView<const Matrix&, false>(*this); }
    auto row(Index i) { return Block<Matrix>(this, i, 0, 1, cols()); }
    auto row(Index i) const { return Block<const Matrix>(this, i, 0, 1, cols()); }
    auto col(Index j) { return Block<Matrix>(this, 0, j, rows(), 1); }
    auto col(Index j) const { return Block<const Matrix>(this, 0, j, rows(), 1); }
    auto leftCols(Index n) { return Block<Matrix>(this, 0, 0, rows(), n); }
    auto leftCols(Index n) const { return Block<const Matrix>(this, 0, 0, rows(), n); }
    auto rightCols(Index n) { return Block<Matrix>(this, 0, cols() - n, rows(), n); }
    auto rightCols(Index n) const { return Block<const Matrix>(this, 0, cols() - n, rows(), n); }
    auto rowwise() { return RowwiseOp<Matrix&>(*this); }
    auto rowwise() const { return RowwiseOp<const Matrix&>(*this); }

    static Matrix Zero() { Matrix m; m.setZero(); return m; }
    static Matrix Zero(Index n) { Matrix m; m.setZero(n); return m; }
    static Matrix Zero(Index r, Index c) { Matrix m; m.setZero(r, c); return m; }
    static Matrix Ones() { Matrix m; m.setOnes(); return m; }
    static Matrix Identity() {
        Matrix m;
        m.setZero();
        for (Index i = 0; i < std::min(m.rows(), m.cols()); ++i) m.coeffRef(i, i) = S(1);
        return m;
    }

private:
    template <class, int, int, int, int, int> friend class Matrix;
    internal::DenseStorage<S, R, C> st_;
};

// array()/matrix() views: same coefficients, different operator* semantics
template <class X, bool A>
struct KindView : std::conditional_t<!std::is_const_v<std::remove_reference_t<X>> && std::is_reference_v<X>,
                                     WritableBase<KindView<X, A>>, DenseBase<KindView<X, A>>> {
    using XT = std::remove_cvref_t<X>;
    using Scalar = typename XT::Scalar;
    static constexpr bool is_array = A;
    static constexpr bool row_major = XT::row_major;
    X x;
    explicit KindView(X v) : x(v) {}
    SVN_EI Index rows() const { return x.rows(); }
    SVN_EI Index cols() const { return x.cols(); }
    SVN_EI Scalar coeff(Index i, Index j) const { return x.coeff(i, j); }
    SVN_EI Scalar& coeffRef(Index i, Index j) { return x.coeffRef(i, j); }
    auto rowwise() { if constexpr (std::is_reference_v<X>) return RowwiseOp<KindView&>(*this); else return RowwiseOp<KindView>(*this); }
    auto rowwise() const { return RowwiseOp<KindView>(*this); }
    template <class E> KindView& operator=(const DenseBase<E>& e) {
        // evaluate first (the right-hand side may read the destination at other coefficients)
        Matrix<Scalar, Dynamic, Dynamic> tmp(e);
        this->assign_loop(tmp, [](auto& a, auto b) SVN_EIL { a = b; });
        return *this;
    }
};

template <class X>
struct Block : std::conditional_t<std::is_const_v<X>, DenseBase<Block<X>>, WritableBase<Block<X>>> {
    using Scalar = typename std::remove_cv_t<X>::Scalar;
    static constexpr bool is_array = false;
    static constexpr bool row_major = std::remove_cv_t<X>::row_major;
    X* m;
    Index i0, j0, r, c;
    Block(X* mm, Index i, Index j, Index rr, Index cc) : m(mm), i0(i), j0(j), r(rr), c(cc) {}
    SVN_EI Index rows() const { return r; }
    SVN_EI Index cols() const { return c; }
    SVN_EI Scalar coeff(Index i, Index j) const { return m->coeff(i0 + i, j0 + j); }
    SVN_EI Scalar& coeffRef(Index i, Index j) { return m->coeffRef(i0 + i, j0 + j); }
    template <class E> Block& operator=(const DenseBase<E>& e) {
        Matrix<Scalar, Dynamic, Dynamic> tmp(e);
        this->assign_loop(tmp, [](auto& a, auto b) SVN_EIL { a = b; });
        return *this;
    }
};

template <class X>
struct Transpose : DenseBase<Transpose<X>> {
    using XT = std::remove_cvref_t<X>;
    using Scalar = typename XT::Scalar;
    static constexpr bool is_array = XT::is_array;
    static constexpr bool row_major = !XT::row_major;
    X x;
    explicit Transpose(const XT& v) : x(v) {}
    SVN_EI Index rows() const { return x.cols(); }
    SVN_EI Index cols() const { return x.rows(); }
    SVN_EI Scalar coeff(Index i, Index j) const { return x.coeff(j, i); }
};

template <class F, class X>
struct CwiseUnaryOp : DenseBase<CwiseUnaryOp<F, X>> {
    using XT = std::remove_cvref_t<X>;
    using Scalar = std::decay_t<decltype(std::declval<F>()(std::declval<typename XT::Scalar>()))>;
    static constexpr bool is_array = XT::is_array;
    static constexpr bool row_major = XT::row_major;
    X x;
    F f;
    CwiseUnaryOp(const XT& v, F ff) : x(v), f(ff) {}
    SVN_EI Index rows() const { return x.rows(); }
    SVN_EI Index cols() const { return x.cols(); }
    SVN_EI Scalar coeff(Index i, Index j) const { return f(x.coeff(i, j)); }
};

template <class F, class L, class R>
struct CwiseBinaryOp : DenseBase<CwiseBinaryOp<F, L, R>> {
    using LT = std::remove_cvref_t<L>;
    using RT = std::remove_cvref_t<R>;
    using Scalar = std::decay_t<decltype(std::declval<F>()(std::declval<typename LT::Scalar>(),
                                                           std::declval<typename RT::Scalar>()))>;
    static constexpr bool is_array = LT::is_array;
    static constexpr bool row_major = LT::row_major;
    L l;
    R r;
    CwiseBinaryOp(const LT& a, const RT& b) : l(a), r(b) {
        if (a.rows() != b.rows() || a.cols() != b.cols())
            throw std::invalid_argument("svn eigen subset: size mismatch in coefficient-wise op");
    }
    SVN_EI Index rows() const { return l.rows(); }
    SVN_EI Index cols() const { return l.cols(); }
    SVN_EI Scalar coeff(Index i, Index j) const { return F{}(l.coeff(i, j), r.coeff(i, j)); }
};

// a row vector repeated over `rows` rows (the right operand of .rowwise() ops)
template <class X>
struct RowBroadcast : DenseBase<RowBroadcast<X>> {
    using XT = std::remove_cvref_t<X>;
    using Scalar = typename XT::Scalar;
    static constexpr bool is_array = XT::is_array;
    static constexpr bool row_major = false;
    X x;
    Index r;
    RowBroadcast(const XT& v, Index rows) : x(v), r(rows) {}
    SVN_EI Index rows() const { return r; }
    SVN_EI Index cols() const { return x.size(); }
    SVN_EI Scalar coeff(Index, Index j) const { return x.vcoeff(j); }
};

template <class X>
struct RowwiseOp {
    using XT = std::remove_cvref_t<X>;
    X x;
    explicit RowwiseOp(X v) : x(v) {}
    template <class V> auto bc(const DenseBase<V>& v) const {
        return RowBroadcast<internal::nested<V>>(v.derived(), x.rows());
    }
    template <class V> auto operator-(const DenseBase<V>& v) const {
        return CwiseBinaryOp<internal::op_diff, internal::nested<XT>, decltype(bc(v))>(x, bc(v));
    }
    template <class V> auto operator+(const DenseBase<V>& v) const {
        return CwiseBinaryOp<internal::op_sum, internal::nested<XT>, decltype(bc(v))>(x, bc(v));
    }
    template <class V> auto operator*(const DenseBase<V>& v) const {
        static_assert(XT::is_array, "rowwise() * needs array operands");
        return CwiseBinaryOp<internal::op_prod, internal::nested<XT>, decltype(bc(v))>(x, bc(v));
    }
    template <class V> void operator+=(const DenseBase<V>& v) { x += bc(v); }
    template <class V> void operator-=(const DenseBase<V>& v) { x -= bc(v); }
    template <class V> void operator*=(const DenseBase<V>& v) { x *= bc(v); }
};

template <class X>
struct ColwiseOp {
    using XT = std::remove_cvref_t<X>;
    using S = typename XT::Scalar;
    X x;
    explicit ColwiseOp(X v) : x(v) {}
    Matrix<S, 1, Dynamic> sum() const {
        Matrix<S, 1, Dynamic> out(x.cols());
        for (Index j = 0; j < x.cols(); ++j)
            out[j] = internal::redux<S>(x.rows(), [&](Index i) SVN_EIL { return x.coeff(i, j); });
        return out;
    }
    Matrix<S, 1, Dynamic> mean() const {
        Matrix<S, 1, Dynamic> out = sum();
        for (Index j = 0; j < x.cols(); ++j) out[j] = out[j] / static_cast<S>(x.rows());
        return out;
    }
};

// ------------------------------------------------------------------------------------------
// Operators
template <internal::Expr A, internal::Expr B>
auto operator+(const A& a, const B& b) {
    internal::check_same_kind<A, B>();
    return CwiseBinaryOp<internal::op_sum, internal::nested<A>, internal::nested<B>>(a, b);
}
template <internal::Expr A, internal::Expr B>
auto operator-(const A& a, const B& b) {
    internal::check_same_kind<A, B>();
    return CwiseBinaryOp<internal::op_diff, internal::nested<A>, internal::nested<B>>(a, b);
}
template <internal::Expr A>
auto operator-(const A& a) { return a.unary(internal::op_neg{}); }

// matrix product, evaluated eagerly (k ascending)
template <class A, class B>
Matrix<typename A::Scalar, Dynamic, Dynamic> product(const A& a, const B& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("svn eigen subset: product size mismatch");
    Matrix<typename A::Scalar, Dynamic, Dynamic> out(a.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) {
            typename A::Scalar acc = 0;
            for (Index k = 0; k < a.cols(); ++k) acc = acc + a.coeff(i, k) * b.coeff(k, j);
            out.coeffRef(i, j) = acc;
        }
    return out;
}
template <internal::Expr A, internal::Expr B>
auto operator*(const A& a, const B& b) {
    internal::check_same_kind<A, B>();
    if constexpr (A::is_array)
        return CwiseBinaryOp<internal::op_prod, internal::nested<A>, internal::nested<B>>(a, b);
    else
        return product(a, b);
}
template <internal::Expr A, internal::Expr B>
auto operator/(const A& a, const B& b) {
    static_assert(A::is_array && B::is_array, "coefficient-wise quotient needs arrays");
    return CwiseBinaryOp<internal::op_quot, internal::nested<A>, internal::nested<B>>(a, b);
}
template <internal::Expr A>
auto operator*(const A& a, const typename A::Scalar& s) { return a.unary(internal::op_scal_r<typename A::Scalar>{s}); }
template <internal::Expr A>
auto operator*(const typename A::Scalar& s, const A& a) { return a.unary(internal::op_scal_l<typename A::Scalar>{s}); }
template <internal::Expr A>
auto operator/(const A& a, const typename A::Scalar& s) { return a.unary(internal::op_div_s<typename A::Scalar>{s}); }
template <internal::Expr A>
auto operator+(const A& a, const typename A::Scalar& s) requires A::is_array {
    return a.unary(internal::op_add_s<typename A::Scalar>{s});
}
template <internal::Expr A>
auto operator-(const A& a, const typename A::Scalar& s) requires A::is_array {
    return a.unary(internal::op_sub_s<typename A::Scalar>{s});
}
#define SVN_EIGEN_CMP(OP, FN, FS)                                                                     \
    template <internal::Expr A, internal::Expr B>                                                     \
    auto operator OP(const A& a, const B& b) requires(A::is_array && B::is_array) {                   \
        return CwiseBinaryOp<internal::FN, internal::nested<A>, internal::nested<B>>(a, b);           \
    }                                                                                                 \
    template <internal::Expr A>                                                                       \
    auto operator OP(const A& a, const typename A::Scalar& s) requires A::is_array {                  \
        return a.unary(internal::FS<typename A::Scalar>{s});                                          \
    }
SVN_EIGEN_CMP(>=, op_ge, op_cmp_ge_s)
SVN_EIGEN_CMP(<=, op_le, op_cmp_le_s)
SVN_EIGEN_CMP(>, op_gt, op_cmp_gt_s)
SVN_EIGEN_CMP(<, op_lt, op_cmp_lt_s)
#undef SVN_EIGEN_CMP

template <class D>
template <class O>
auto DenseBase<D>::cross(const DenseBase<O>& o) const {
    const D& a = derived();
    const O& b = o.derived();
    return Matrix<typename D::Scalar, 3, 1>(a.vcoeff(1) * b.vcoeff(2) - a.vcoeff(2) * b.vcoeff(1),
                                            a.vcoeff(2) * b.vcoeff(0) - a.vcoeff(0) * b.vcoeff(2),
                                            a.vcoeff(0) * b.vcoeff(1) - a.vcoeff(1) * b.vcoeff(0));
}
template <class D>
auto DenseBase<D>::unitOrthogonal() const {
    // a unit vector orthogonal to this 3-vector (choice of Eigen's documented construction:
    // drop the coordinate of largest magnitude's partner)
    using S = typename D::Scalar;
    const S x0 = vcoeff(0), y0 = vcoeff(1), z0 = vcoeff(2);
    if (std::abs(x0) > std::abs(z0) || std::abs(y0) > std::abs(z0)) {
        const S inv = S(1) / std::sqrt(x0 * x0 + y0 * y0);
        return Matrix<S, 3, 1>(-y0 * inv, x0 * inv, S(0));
    }
    const S inv = S(1) / std::sqrt(y0 * y0 + z0 * z0);
    return Matrix<S, 3, 1>(S(0), -z0 * inv, y0 * inv);
}

// ------------------------------------------------------------------------------------------
using MatrixXf = Matrix<float, Dynamic, Dynamic>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXf = Matrix<float, Dynamic, 1>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXf = Matrix<float, 1, Dynamic>;
using Vector3f = Matrix<float, 3, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector3i = Matrix<int, 3, 1>;
using Matrix3d = Matrix<double, 3, 3>;
static_assert(sizeof(Vector3d) == 3 * sizeof(double), "fixed-size storage must be inline (Eigen layout)");

}  // namespace Eigen
