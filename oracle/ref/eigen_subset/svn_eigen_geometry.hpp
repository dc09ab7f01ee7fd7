// svn_eigen_geometry.hpp — TEST INFRASTRUCTURE ONLY.  The Eigen/Geometry types the
// reference's headers and src/robot.cpp use (Quaternion, AngleAxis, Translation, Isometry
// transforms), written independently on top of svn_eigen_subset.hpp.  Only the nn path's
// numerics are pinned through this build; these exist so the unmodified translation units
// compile (robot.cpp supplies RobotModel::reach() for make_normalizer, nn.cpp:324).
#pragma once
#include "svn_eigen_subset.hpp"

namespace Eigen {

template <class S> using Vec3T = Matrix<S, 3, 1>;
template <class S> using Mat3T = Matrix<S, 3, 3>;

template <class S>
Vec3T<S> mat3_vec(const Mat3T<S>& m, const Vec3T<S>& v) {
    Vec3T<S> o;
    for (int i = 0; i < 3; ++i) o[i] = m.coeff(i, 0) * v[0] + m.coeff(i, 1) * v[1] + m.coeff(i, 2) * v[2];
    return o;
}
template <class S>
Mat3T<S> mat3_mul(const Mat3T<S>& a, const Mat3T<S>& b) {
    Mat3T<S> o;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.coeffRef(i, j) = a.coeff(i, 0) * b.coeff(0, j) + a.coeff(i, 1) * b.coeff(1, j) + a.coeff(i, 2) * b.coeff(2, j);
    return o;
}

template <class S>
struct Quaternion {
    S w_ = 1, x_ = 0, y_ = 0, z_ = 0;
    Quaternion() = default;
    Quaternion(S w, S x, S y, S z) : w_(w), x_(x), y_(y), z_(z) {}
    explicit Quaternion(const Mat3T<S>& m) {  // rotation matrix -> unit quaternion (trace method)
        const S t = m.coeff(0, 0) + m.coeff(1, 1) + m.coeff(2, 2);
        if (t > 0) {
            const S r = std::sqrt(t + 1), s = S(0.5) / r;
            w_ = S(0.5) * r;
            x_ = (m.coeff(2, 1) - m.coeff(1, 2)) * s;
            y_ = (m.coeff(0, 2) - m.coeff(2, 0)) * s;
            z_ = (m.coeff(1, 0) - m.coeff(0, 1)) * s;
        } else {
            int i = 0;
            if (m.coeff(1, 1) > m.coeff(0, 0)) i = 1;
            if (m.coeff(2, 2) > m.coeff(i, i)) i = 2;
            const int j = (i + 1) % 3, k = (j + 1) % 3;
            const S r = std::sqrt(m.coeff(i, i) - m.coeff(j, j) - m.coeff(k, k) + 1), s = S(0.5) / r;
            S q[3];
            q[i] = S(0.5) * r;
            q[j] = (m.coeff(j, i) + m.coeff(i, j)) * s;
            q[k] = (m.coeff(k, i) + m.coeff(i, k)) * s;
            w_ = (m.coeff(k, j) - m.coeff(j, k)) * s;
            x_ = q[0], y_ = q[1], z_ = q[2];
        }
    }
    S w() const { return w_; }
    S x() const { return x_; }
    S y() const { return y_; }
    S z() const { return z_; }
    S norm() const { return std::sqrt(w_ * w_ + x_ * x_ + y_ * y_ + z_ * z_); }
    Quaternion normalized() const {
        const S n = norm();
        return {w_ / n, x_ / n, y_ / n, z_ / n};
    }
    Mat3T<S> toRotationMatrix() const {
        Mat3T<S> r;
        const S w = w_, x = x_, y = y_, z = z_;
        r.coeffRef(0, 0) = 1 - 2 * (y * y + z * z);
        r.coeffRef(0, 1) = 2 * (x * y - z * w);
        r.coeffRef(0, 2) = 2 * (x * z + y * w);
        r.coeffRef(1, 0) = 2 * (x * y + z * w);
        r.coeffRef(1, 1) = 1 - 2 * (x * x + z * z);
        r.coeffRef(1, 2) = 2 * (y * z - x * w);
        r.coeffRef(2, 0) = 2 * (x * z - y * w);
        r.coeffRef(2, 1) = 2 * (y * z + x * w);
        r.coeffRef(2, 2) = 1 - 2 * (x * x + y * y);
        return r;
    }
};

template <class S>
struct AngleAxis {
    S angle;
    Vec3T<S> axis;
    AngleAxis(S a, const Vec3T<S>& ax) : angle(a), axis(ax) {}
    Mat3T<S> toRotationMatrix() const {  // Rodrigues
        const S c = std::cos(angle), s = std::sin(angle), t = 1 - c;
        const S x = axis[0], y = axis[1], z = axis[2];
        Mat3T<S> r;
        r.coeffRef(0, 0) = t * x * x + c;
        r.coeffRef(0, 1) = t * x * y - s * z;
        r.coeffRef(0, 2) = t * x * z + s * y;
        r.coeffRef(1, 0) = t * x * y + s * z;
        r.coeffRef(1, 1) = t * y * y + c;
        r.coeffRef(1, 2) = t * y * z - s * x;
        r.coeffRef(2, 0) = t * x * z - s * y;
        r.coeffRef(2, 1) = t * y * z + s * x;
        r.coeffRef(2, 2) = t * z * z + c;
        return r;
    }
};

template <class S, int Dim>
struct Translation {
    Vec3T<S> v;
    explicit Translation(const Vec3T<S>& t) : v(t) {}
};

enum TransformTraits { Isometry = 1, Affine = 2 };

template <class S, int Dim, int Mode>
struct Transform {
    Mat3T<S> lin = Mat3T<S>::Identity();
    Vec3T<S> tr = Vec3T<S>::Zero();
    static Transform Identity() { return Transform(); }
    Mat3T<S>& linear() { return lin; }
    const Mat3T<S>& linear() const { return lin; }
    Vec3T<S>& translation() { return tr; }
    const Vec3T<S>& translation() const { return tr; }
    Transform operator*(const AngleAxis<S>& a) const {
        Transform o = *this;
        o.lin = mat3_mul(lin, a.toRotationMatrix());
        return o;
    }
    Transform operator*(const Translation<S, Dim>& t) const {
        Transform o = *this;
        const Vec3T<S> d = mat3_vec(lin, t.v);
        for (int i = 0; i < 3; ++i) o.tr[i] = tr[i] + d[i];
        return o;
    }
    Transform operator*(const Transform& b) const {
        Transform o;
        o.lin = mat3_mul(lin, b.lin);
        const Vec3T<S> d = mat3_vec(lin, b.tr);
        for (int i = 0; i < 3; ++i) o.tr[i] = tr[i] + d[i];
        return o;
    }
    Vec3T<S> operator*(const Vec3T<S>& p) const {
        Vec3T<S> d = mat3_vec(lin, p);
        for (int i = 0; i < 3; ++i) d[i] = d[i] + tr[i];
        return d;
    }
};

using Quaterniond = Quaternion<double>;
using AngleAxisd = AngleAxis<double>;
using Translation3d = Translation<double, 3>;
using Isometry3d = Transform<double, 3, Isometry>;

}  // namespace Eigen
