#pragma once
// fskin-b200 — reference-facing C++ API (drop-in for proj/include/fskin/geometry.hpp).
//
// The reference aliases Eigen fixed-size types (geometry.hpp:9-11). Eigen is not a
// dependency here: Vec3 / Mat3 / Mat34 are small value types exposing the subset of the
// Eigen interface the deformer/correspondence API and its callers use (x()/y()/z(),
// operator(), Zero/Identity/UnitX, dot/norm/cross, transpose/determinant/inverse).

#include <algorithm>
#include <cmath>
#include <limits>

namespace fskin {

struct Vec3 {
    double v[3] = {0.0, 0.0, 0.0};

    Vec3() = default;
    Vec3(double x, double y, double z) : v{x, y, z} {}

    static Vec3 Zero() { return {}; }
    static Vec3 Ones() { return {1.0, 1.0, 1.0}; }
    static Vec3 Constant(double c) { return {c, c, c}; }
    static Vec3 UnitX() { return {1.0, 0.0, 0.0}; }
    static Vec3 UnitY() { return {0.0, 1.0, 0.0}; }
    static Vec3 UnitZ() { return {0.0, 0.0, 1.0}; }

    double& x() { return v[0]; }
    double& y() { return v[1]; }
    double& z() { return v[2]; }
    double x() const { return v[0]; }
    double y() const { return v[1]; }
    double z() const { return v[2]; }
    double& operator()(int i) { return v[i]; }
    double operator()(int i) const { return v[i]; }
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    double* data() { return v; }
    const double* data() const { return v; }
    static constexpr int size() { return 3; }

    Vec3 operator+(const Vec3& o) const { return {v[0] + o.v[0], v[1] + o.v[1], v[2] + o.v[2]}; }
    Vec3 operator-(const Vec3& o) const { return {v[0] - o.v[0], v[1] - o.v[1], v[2] - o.v[2]}; }
    Vec3 operator-() const { return {-v[0], -v[1], -v[2]}; }
    Vec3 operator*(double s) const { return {v[0] * s, v[1] * s, v[2] * s}; }
    Vec3 operator/(double s) const { return {v[0] / s, v[1] / s, v[2] / s}; }
    Vec3& operator+=(const Vec3& o) { v[0] += o.v[0]; v[1] += o.v[1]; v[2] += o.v[2]; return *this; }
    Vec3& operator-=(const Vec3& o) { v[0] -= o.v[0]; v[1] -= o.v[1]; v[2] -= o.v[2]; return *this; }
    Vec3& operator*=(double s) { v[0] *= s; v[1] *= s; v[2] *= s; return *this; }
    bool operator==(const Vec3& o) const { return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2]; }

    double dot(const Vec3& o) const { return v[0] * o.v[0] + v[1] * o.v[1] + v[2] * o.v[2]; }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    Vec3 normalized() const { const double n = norm(); return n > 0 ? *this / n : *this; }
    Vec3 cross(const Vec3& o) const {
        return {v[1] * o.v[2] - v[2] * o.v[1], v[2] * o.v[0] - v[0] * o.v[2], v[0] * o.v[1] - v[1] * o.v[0]};
    }
    Vec3 cwiseMin(const Vec3& o) const { return {std::min(v[0], o.v[0]), std::min(v[1], o.v[1]), std::min(v[2], o.v[2])}; }
    Vec3 cwiseMax(const Vec3& o) const { return {std::max(v[0], o.v[0]), std::max(v[1], o.v[1]), std::max(v[2], o.v[2])}; }
};

inline Vec3 operator*(double s, const Vec3& a) { return a * s; }

struct Mat3 {
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};

    static Mat3 Zero() { return {}; }
    static Mat3 Identity() {
        Mat3 r;
        r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
        return r;
    }
    double& operator()(int r, int c) { return m[r][c]; }
    double operator()(int r, int c) const { return m[r][c]; }

    Mat3 transpose() const {
        Mat3 t;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) t.m[i][j] = m[j][i];
        return t;
    }
    // Closed-form cofactor expansion (what Eigen does for 3x3).
    double determinant() const {
        return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
               m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
    }
    Mat3 inverse() const {
        Mat3 c;
        c.m[0][0] = m[1][1] * m[2][2] - m[1][2] * m[2][1];
        c.m[0][1] = m[0][2] * m[2][1] - m[0][1] * m[2][2];
        c.m[0][2] = m[0][1] * m[1][2] - m[0][2] * m[1][1];
        c.m[1][0] = m[1][2] * m[2][0] - m[1][0] * m[2][2];
        c.m[1][1] = m[0][0] * m[2][2] - m[0][2] * m[2][0];
        c.m[1][2] = m[0][2] * m[1][0] - m[0][0] * m[1][2];
        c.m[2][0] = m[1][0] * m[2][1] - m[1][1] * m[2][0];
        c.m[2][1] = m[0][1] * m[2][0] - m[0][0] * m[2][1];
        c.m[2][2] = m[0][0] * m[1][1] - m[0][1] * m[1][0];
        const double inv = 1.0 / (m[0][0] * c.m[0][0] + m[0][1] * c.m[1][0] + m[0][2] * c.m[2][0]);
        for (auto& row : c.m)
            for (double& e : row) e *= inv;
        return c;
    }
    Vec3 operator*(const Vec3& x) const {
        return {m[0][0] * x[0] + m[0][1] * x[1] + m[0][2] * x[2], m[1][0] * x[0] + m[1][1] * x[1] + m[1][2] * x[2],
                m[2][0] * x[0] + m[2][1] * x[1] + m[2][2] * x[2]};
    }
    Mat3 operator*(const Mat3& b) const {
        Mat3 r;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) r.m[i][j] = m[i][0] * b.m[0][j] + m[i][1] * b.m[1][j] + m[i][2] * b.m[2][j];
        return r;
    }
    Mat3 operator*(double s) const {
        Mat3 r = *this;
        for (auto& row : r.m)
            for (double& e : row) e *= s;
        return r;
    }
    Mat3 operator+(const Mat3& b) const {
        Mat3 r = *this;
        r += b;
        return r;
    }
    Mat3& operator+=(const Mat3& b) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m[i][j] += b.m[i][j];
        return *this;
    }
    double norm() const {
        double s = 0.0;
        for (const auto& row : m)
            for (double e : row) s += e * e;
        return std::sqrt(s);
    }
};

inline Mat3 operator*(double s, const Mat3& a) { return a * s; }

/// 3x4 [linear | translation], row-major.
struct Mat34 {
    double m[3][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
    double& operator()(int r, int c) { return m[r][c]; }
    double operator()(int r, int c) const { return m[r][c]; }
};

/// Axis-aligned box in canonical or posed space (geometry.hpp:14-39).
struct Aabb {
    Vec3 min = Vec3::Zero();
    Vec3 max = Vec3::Ones();

    static Aabb empty() {
        const double inf = std::numeric_limits<double>::infinity();
        return {Vec3::Constant(inf), Vec3::Constant(-inf)};
    }
    Vec3 extent() const { return max - min; }
    double diagonal() const { return extent().norm(); }
    bool contains(const Vec3& p) const {
        for (int a = 0; a < 3; ++a)
            if (!(p[a] >= min[a] && p[a] <= max[a])) return false;
        return true;
    }
    Vec3 clamp(const Vec3& p) const { return p.cwiseMax(min).cwiseMin(max); }
    Aabb padded(double margin) const { return {min - Vec3::Constant(margin), max + Vec3::Constant(margin)}; }
    void expand(const Vec3& p) {
        min = min.cwiseMin(p);
        max = max.cwiseMax(p);
    }
};

/// Rigid body motion [R | t] (geometry.hpp:42-78).
struct RigidTransform {
    Mat3 rotation = Mat3::Identity();
    Vec3 translation = Vec3::Zero();

    static RigidTransform identity() { return {}; }
    /// Rotation by `angle` radians about the line through `pivot` with direction `axis`
    /// (geometry.cpp:7-14; Rodrigues).
    static RigidTransform about_axis(const Vec3& pivot, const Vec3& axis, double angle);

    Vec3 apply(const Vec3& x) const { return rotation * x + translation; }
    RigidTransform compose(const RigidTransform& rhs) const {
        return {rotation * rhs.rotation, rotation * rhs.translation + translation};
    }
    RigidTransform inverse() const {
        const Mat3 rt = rotation.transpose();
        return {rt, -(rt * translation)};
    }
    double orthonormality_error() const {
        Mat3 d = rotation.transpose() * rotation;
        d += Mat3::Identity() * -1.0;
        return d.norm();
    }
    bool is_rigid(double tol = 1e-6) const { return orthonormality_error() <= tol && rotation.determinant() > 0.0; }
    Mat34 matrix() const {
        Mat34 o;
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) o.m[r][c] = rotation.m[r][c];
            o.m[r][3] = translation[r];
        }
        return o;
    }
};

inline RigidTransform operator*(const RigidTransform& a, const RigidTransform& b) { return a.compose(b); }
inline RigidTransform invert(const RigidTransform& t) { return t.inverse(); }
inline Vec3 apply(const RigidTransform& t, const Vec3& x) { return t.apply(x); }

/// General affine 3x4 map (geometry.hpp:90-112).
struct Affine3 {
    Mat3 linear = Mat3::Identity();
    Vec3 translation = Vec3::Zero();

    static Affine3 zero() { return {Mat3::Zero(), Vec3::Zero()}; }
    static Affine3 from(const RigidTransform& t) { return {t.rotation, t.translation}; }
    Vec3 apply(const Vec3& x) const { return linear * x + translation; }
    Affine3& operator+=(const Affine3& o) {
        linear += o.linear;
        translation += o.translation;
        return *this;
    }
    Affine3 operator*(double s) const { return {linear * s, translation * s}; }
    Mat34 matrix() const {
        Mat34 o;
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) o.m[r][c] = linear.m[r][c];
            o.m[r][3] = translation[r];
        }
        return o;
    }
};

/// Distance from p to the segment [a, b] (geometry.cpp:17-23).
double point_segment_distance(const Vec3& p, const Vec3& a, const Vec3& b);

}  // namespace fskin
