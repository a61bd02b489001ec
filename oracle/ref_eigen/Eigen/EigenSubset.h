// TEST INFRASTRUCTURE ONLY — never part of the product.
//
// A restatement of the subset of Eigen 3.4.0 that the reference's hot path uses
// (/root/reference/proj/CMakeLists.txt:10 pins Eigen3 >= 3.3; Ubuntu 24.04 ships 3.4.0; Eigen is
// not vendored and not installed here, so the reference cannot be built against the real
// library). It exists so that oracle/ref_build.sh can compile the reference's own sources
// UNCHANGED (oracle/_ref/libgsref.so) and pin the oracle restatement against them.
//
// Only fixed-size double matrices up to 4x4, quaternions and angle-axis rotations are covered.
// Everything is evaluated eagerly; that is exact for element-wise expressions (each coefficient
// sees the same operations in the same order; the reference's build has no FMA: x86-64 without
// -march). What Eigen decides — and what this file restates — is the ORDER of the sums inside
// products, dot products and reductions, for an SSE2 build (packets of 2 doubles,
// EIGEN_UNALIGNED_VECTORIZE = 1, complete unrolling of fixed sizes):
//
//  * redux (sum(), dot(), squaredNorm(), the inner sum of a coefficient-based product):
//      - when the reduced expression has packet access (contiguous operands): the packets
//        (e0,e1), (e2,e3), ... are added as a halving tree of packets, the packet is summed
//        lane0 + lane1, and an odd last element is added after (Redux.h, redux_vec_unroller +
//        LinearVectorizedTraversal): 3 terms (e0+e1)+e2, 4 terms (e0+e2)+(e1+e3);
//      - otherwise (strided operands: a row of a column-major matrix, a diagonal): a halving
//        tree of scalars (redux_novec_unroller): 3 terms e0+(e1+e2), 4 terms (e0+e1)+(e2+e3).
//  * small products (all dimensions fixed and small: coefficient-based "lazy" products,
//    ProductEvaluators.h): the product has packet access when its lhs is column-major (not a
//    transpose) and has more than one row (CanVectorizeLhs), or its rhs is row-major with more
//    than one column (CanVectorizeRhs); it evaluates row-major only for row vectors or when the
//    rhs is row-major and the lhs cannot vectorise. A destination whose storage order agrees
//    is assigned with packets of 2 along its inner dimension (inner / linear / slice
//    vectorised traversal): those coefficients are the sequential sum over k
//    (etor_product_packet_impl: pmul, then pmadd = mul + add in k order); a leftover odd
//    coefficient, or every coefficient when the product has no packet access, is the redux of
//    lhs.row(i) .* rhs.col(j) above.
//  * products with a depth of 1 are outer products (one multiplication per coefficient).
//  * quaternions: q * v = v + w uv + vec x uv with uv = 2 (vec x v) (Quaternion.h,
//    _transformVector); toRotationMatrix from tx = 2x, ...; coefficients stored (x, y, z, w).
//  * 2x2 inverse = adjugate * (1 / det), det = a00 a11 - a10 a01 (InverseImpl.h).
//
// Known deviation: Eigen vectorises array().exp() with its own Cephes-style pexp on the packet
// lanes (elements 0 and 1 of a 3-vector); this file calls std::exp on every element, so
// exp-derived values may differ from a real Eigen build by an ulp (the tolerance the parity
// tests state where exp enters).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstddef>
#include <type_traits>

namespace Eigen {

using Index = std::ptrdiff_t;
enum { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };

namespace internal {

// unvectorised complete-unrolled reduction: halving tree
inline double redux_novec(const double* e, int n) {
    if (n == 1) return e[0];
    const int h = n / 2;
    return redux_novec(e, h) + redux_novec(e + h, n - h);
}

// packets of 2 combined as a halving tree of packets
inline void redux_vec_packets(const double* e, int np, double out[2]) {
    if (np == 1) {
        out[0] = e[0];
        out[1] = e[1];
        return;
    }
    const int h = np / 2;
    double a[2], b[2];
    redux_vec_packets(e, h, a);
    redux_vec_packets(e + 2 * h, np - h, b);
    out[0] = a[0] + b[0];
    out[1] = a[1] + b[1];
}

// vectorised reduction (LinearVectorizedTraversal, complete unrolling)
inline double redux_vec(const double* e, int n) {
    const int np = n / 2;
    if (np == 0) return redux_novec(e, n);
    double p[2];
    redux_vec_packets(e, np, p);
    double r = p[0] + p[1];
    if (n % 2) r = r + redux_novec(e + 2 * np, n - 2 * np);
    return r;
}

}  // namespace internal

template <typename Scalar, int R, int C, int Options = 0, int MaxR = R, int MaxC = C>
class Matrix;
template <int R, int C>
class TransposeRef;
template <int N>
class DiagonalMatrix;
template <int R, int C>
class ArrayVal;

template <int R, int C, bool Const>
class ArrayRef;

namespace internal {

// Coefficient-based product of a logical R x K lhs and K x C rhs (see the header comment).
// lhs_rm / rhs_rm: the operand is a row-major view (a transpose of a column-major matrix).
template <int R, int K, int C, class LA, class RA>
void lazy_product(const LA& a, bool lhs_rm, const RA& b, bool rhs_rm, double* out /* col-major R x C */) {
    const bool can_lhs = !lhs_rm && R != 1;
    const bool can_rhs = rhs_rm && C != 1;
    const bool eval_rm = (R == 1 && C != 1) ? true : (C == 1 && R != 1) ? false : (rhs_rm && !can_lhs);
    const bool dst_rm = (R == 1 && C != 1);
    const bool vec = (can_lhs || can_rhs) && (dst_rm == eval_rm);
    // redux of lhs.row(i) .* rhs.col(j): packet access iff both are contiguous
    const bool redux_packet = (lhs_rm || R == 1) && (!rhs_rm || C == 1);
    auto coeff = [&](int i, int j) {
        double e[K];
        for (int k = 0; k < K; ++k) e[k] = a(i, k) * b(k, j);
        return redux_packet ? redux_vec(e, K) : redux_novec(e, K);
    };
    auto seq = [&](int i, int j) {
        double s = a(i, 0) * b(0, j);
        for (int k = 1; k < K; ++k) s = s + a(i, k) * b(k, j);
        return s;
    };
    for (int j = 0; j < C; ++j)
        for (int i = 0; i < R; ++i) {
            double v;
            if (!vec) v = coeff(i, j);
            else if (!dst_rm) v = i < 2 * (R / 2) ? seq(i, j) : coeff(i, j);
            else v = j < 2 * (C / 2) ? seq(i, j) : coeff(i, j);
            out[j * R + i] = v;
        }
}

template <int R, int C>
struct CommaInit;

}  // namespace internal

// ------------------------------------------------------------------------------------------
template <typename Scalar, int R, int C, int Options, int MaxR, int MaxC>
class Matrix {
    static_assert(std::is_same<Scalar, double>::value, "EigenSubset: double only");

public:
    static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C, SizeAtCompileTime = R * C;
    double m_d[R * C];  // column-major

    Matrix() {}
    Matrix(double x, double y) {
        static_assert(R * C == 2, "2-vector constructor");
        m_d[0] = x;
        m_d[1] = y;
    }
    Matrix(double x, double y, double z) {
        static_assert(R * C == 3, "3-vector constructor");
        m_d[0] = x;
        m_d[1] = y;
        m_d[2] = z;
    }
    Matrix(double x, double y, double z, double w) {
        static_assert(R * C == 4, "4-vector constructor");
        m_d[0] = x;
        m_d[1] = y;
        m_d[2] = z;
        m_d[3] = w;
    }
    template <int TR, int TC>
    Matrix(const TransposeRef<TR, TC>& t);
    Matrix(const ArrayVal<R, C>& a);

    static Matrix Zero() { return Constant(0.0); }
    // Eigen 3.4 internal::random<double>() = -1 + 2 * rand() / RAND_MAX (random_default_impl),
    // coefficients in storage order (the reference's unit tests draw scenes with it)
    static Matrix Random() {
        Matrix m;
        for (int i = 0; i < R * C; ++i) m.m_d[i] = -1.0 + 2.0 * static_cast<double>(std::rand()) / RAND_MAX;
        return m;
    }
    static Matrix Constant(double v) {
        Matrix m;
        for (int i = 0; i < R * C; ++i) m.m_d[i] = v;
        return m;
    }
    static Matrix Identity() {
        Matrix m = Zero();
        for (int i = 0; i < std::min(R, C); ++i) m(i, i) = 1.0;
        return m;
    }
    static Matrix Unit(int k) {
        Matrix m = Zero();
        m.m_d[k] = 1.0;
        return m;
    }
    static Matrix UnitX() { return Unit(0); }
    static Matrix UnitY() { return Unit(1); }
    static Matrix UnitZ() { return Unit(2); }
    static Matrix UnitW() { return Unit(3); }

    static constexpr Index rows() { return R; }
    static constexpr Index cols() { return C; }
    static constexpr Index size() { return R * C; }
    double* data() { return m_d; }
    const double* data() const { return m_d; }

    double& operator()(Index i, Index j) { return m_d[j * R + i]; }
    double operator()(Index i, Index j) const { return m_d[j * R + i]; }
    double& operator()(Index i) { return m_d[i]; }
    double operator()(Index i) const { return m_d[i]; }
    double& operator[](Index i) { return m_d[i]; }
    double operator[](Index i) const { return m_d[i]; }
    double coeff(Index i, Index j) const { return (*this)(i, j); }
    double coeff(Index i) const { return m_d[i]; }
    double& x() { return m_d[0]; }
    double& y() { return m_d[1]; }
    double& z() { return m_d[2]; }
    double& w() { return m_d[3]; }
    double x() const { return m_d[0]; }
    double y() const { return m_d[1]; }
    double z() const { return m_d[2]; }
    double w() const { return m_d[3]; }

    Matrix& setZero() { return *this = Zero(); }
    Matrix& setConstant(double v) { return *this = Constant(v); }
    Matrix& setOnes() { return *this = Constant(1.0); }
    Matrix& setIdentity() { return *this = Identity(); }

    internal::CommaInit<R, C> operator<<(double v);

    // element-wise
    Matrix operator+(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m_d[i] + o.m_d[i];
        return r;
    }
    Matrix operator-(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m_d[i] - o.m_d[i];
        return r;
    }
    Matrix operator-() const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = -m_d[i];
        return r;
    }
    Matrix operator*(double s) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m_d[i] * s;
        return r;
    }
    Matrix operator/(double s) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m_d[i] / s;
        return r;
    }
    Matrix& operator+=(const Matrix& o) { return *this = *this + o; }
    Matrix& operator-=(const Matrix& o) { return *this = *this - o; }
    Matrix& operator*=(double s) { return *this = *this * s; }
    Matrix& operator/=(double s) { return *this = *this / s; }
    template <int TR, int TC>
    Matrix operator+(const TransposeRef<TR, TC>& t) const {
        return *this + Matrix(t);
    }
    template <int TR, int TC>
    Matrix operator-(const TransposeRef<TR, TC>& t) const {
        return *this - Matrix(t);
    }

    bool operator==(const Matrix& o) const {
        for (int i = 0; i < R * C; ++i)
            if (!(m_d[i] == o.m_d[i])) return false;
        return true;
    }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

    Matrix cwiseMax(double v) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = std::max(m_d[i], v);
        return r;
    }
    Matrix cwiseMin(double v) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = std::min(m_d[i], v);
        return r;
    }
    Matrix cwiseMax(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = std::max(m_d[i], o.m_d[i]);
        return r;
    }
    Matrix cwiseMin(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = std::min(m_d[i], o.m_d[i]);
        return r;
    }
    Matrix cwiseProduct(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m_d[i] * o.m_d[i];
        return r;
    }
    Matrix cwiseAbs() const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = std::abs(m_d[i]);
        return r;
    }

    // reductions over contiguous storage (packet access)
    double sum() const { return internal::redux_vec(m_d, R * C); }
    double dot(const Matrix& o) const {
        double e[R * C];
        for (int i = 0; i < R * C; ++i) e[i] = m_d[i] * o.m_d[i];
        return internal::redux_vec(e, R * C);
    }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    Matrix normalized() const {  // MatrixBase::normalized: n / sqrt(|n|^2) when nonzero
        const double z = squaredNorm();
        return z > 0.0 ? *this / std::sqrt(z) : *this;
    }
    void normalize() { *this = normalized(); }
    double maxCoeff() const { return *std::max_element(m_d, m_d + R * C); }
    double minCoeff() const { return *std::min_element(m_d, m_d + R * C); }
    bool isZero(double prec = 1e-12) const {
        for (int i = 0; i < R * C; ++i)
            if (!(std::abs(m_d[i]) <= prec)) return false;
        return true;
    }
    bool allFinite() const {
        for (int i = 0; i < R * C; ++i)
            if (!std::isfinite(m_d[i])) return false;
        return true;
    }

    Matrix cross(const Matrix& v) const {  // OrthoMethods.h
        static_assert(R * C == 3, "cross of 3-vectors");
        return Matrix(m_d[1] * v.m_d[2] - m_d[2] * v.m_d[1], m_d[2] * v.m_d[0] - m_d[0] * v.m_d[2],
                      m_d[0] * v.m_d[1] - m_d[1] * v.m_d[0]);
    }

    // diagonal: strided (no packet access)
    double trace() const {
        double e[R < C ? R : C];
        for (int i = 0; i < (R < C ? R : C); ++i) e[i] = (*this)(i, i);
        return internal::redux_novec(e, R < C ? R : C);
    }
    double determinant() const {
        static_assert(R == 2 && C == 2, "determinant: 2x2 only");
        return m_d[0] * m_d[3] - m_d[1] * m_d[2];
    }
    Matrix inverse() const {
        static_assert(R == 2 && C == 2, "inverse: 2x2 only");
        const double invdet = 1.0 / determinant();
        Matrix r;
        const double temp = (*this)(0, 0);
        r(0, 0) = (*this)(1, 1) * invdet;
        r(1, 0) = -(*this)(1, 0) * invdet;
        r(0, 1) = -(*this)(0, 1) * invdet;
        r(1, 1) = temp * invdet;
        return r;
    }

    TransposeRef<C, R> transpose() const;
    DiagonalMatrix<R * C> asDiagonal() const;
    struct DiagRef {
        Matrix* m;
        DiagRef& array() { return *this; }
        DiagRef& operator+=(double v) {
            for (int i = 0; i < (R < C ? R : C); ++i) (*m)(i, i) = (*m)(i, i) + v;
            return *this;
        }
        double sum() const { return m->trace(); }
    };
    DiagRef diagonal() { return DiagRef{this}; }
    ArrayRef<R, C, false> array();
    ArrayRef<R, C, true> array() const;
};

template <typename S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC> operator*(double s, const Matrix<S, R, C, O, MR, MC>& m) {
    Matrix<S, R, C, O, MR, MC> r;
    for (int i = 0; i < R * C; ++i) r.m_d[i] = s * m.m_d[i];
    return r;
}

// logical R x C row-major view of a column-major C x R matrix (Transpose<>)
template <int R, int C>
class TransposeRef {
public:
    const Matrix<double, C, R>& m;
    double operator()(Index i, Index j) const { return m(j, i); }
    Matrix<double, R, C> eval() const { return Matrix<double, R, C>(*this); }
    template <int TR, int TC>
    friend class TransposeRef;
};

template <typename S, int R, int C, int O, int MR, int MC>
template <int TR, int TC>
Matrix<S, R, C, O, MR, MC>::Matrix(const TransposeRef<TR, TC>& t) {
    static_assert(TR == R && TC == C, "transpose shape");
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < C; ++j) (*this)(i, j) = t(i, j);
}

template <typename S, int R, int C, int O, int MR, int MC>
TransposeRef<C, R> Matrix<S, R, C, O, MR, MC>::transpose() const {
    return TransposeRef<C, R>{*this};
}

template <int R, int C, int TR, int TC>
Matrix<double, R, C> operator+(const TransposeRef<TR, TC>& t, const Matrix<double, R, C>& m) {
    return Matrix<double, R, C>(t) + m;
}

// ---- products
template <int R, int K, int C>
Matrix<double, R, C> operator*(const Matrix<double, R, K>& a, const Matrix<double, K, C>& b) {
    Matrix<double, R, C> r;
    internal::lazy_product<R, K, C>(a, false, b, false, r.m_d);
    return r;
}
template <int R, int K, int C>
Matrix<double, R, C> operator*(const TransposeRef<R, K>& a, const Matrix<double, K, C>& b) {
    Matrix<double, R, C> r;
    internal::lazy_product<R, K, C>(a, true, b, false, r.m_d);
    return r;
}
template <int R, int K, int C>
Matrix<double, R, C> operator*(const Matrix<double, R, K>& a, const TransposeRef<K, C>& b) {
    Matrix<double, R, C> r;
    internal::lazy_product<R, K, C>(a, false, b, true, r.m_d);
    return r;
}
template <int R, int K, int C>
Matrix<double, R, C> operator*(const TransposeRef<R, K>& a, const TransposeRef<K, C>& b) {
    Matrix<double, R, C> r;
    internal::lazy_product<R, K, C>(a, true, b, true, r.m_d);
    return r;
}
// outer products (depth 1): one multiplication per coefficient
template <int R, int C>
Matrix<double, R, C> operator*(const Matrix<double, R, 1>& a, const TransposeRef<1, C>& b) {
    Matrix<double, R, C> r;
    for (int j = 0; j < C; ++j)
        for (int i = 0; i < R; ++i) r(i, j) = b(0, j) * a(i, 0);
    return r;
}

// diagonal products: coefficient a(i, j) * d(j)
template <int N>
class DiagonalMatrix {
public:
    double d[N];
};
template <typename S, int R, int C, int O, int MR, int MC>
DiagonalMatrix<R * C> Matrix<S, R, C, O, MR, MC>::asDiagonal() const {
    DiagonalMatrix<R * C> r;
    for (int i = 0; i < R * C; ++i) r.d[i] = m_d[i];
    return r;
}
template <int R, int C>
Matrix<double, R, C> operator*(const Matrix<double, R, C>& a, const DiagonalMatrix<C>& d) {
    Matrix<double, R, C> r;
    for (int j = 0; j < C; ++j)
        for (int i = 0; i < R; ++i) r(i, j) = a(i, j) * d.d[j];
    return r;
}

// ---- arrays (coefficient-wise views of plain matrices: packet access)
template <int R, int C>
class ArrayVal {
public:
    double m_d[R * C];
    double sum() const { return internal::redux_vec(m_d, R * C); }
    ArrayVal exp() const {
        ArrayVal r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = std::exp(m_d[i]);
        return r;
    }
    ArrayVal operator*(const ArrayVal& o) const {
        ArrayVal r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m_d[i] * o.m_d[i];
        return r;
    }
    Matrix<double, R, C> matrix() const { return Matrix<double, R, C>(*this); }
};

template <typename S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC>::Matrix(const ArrayVal<R, C>& a) {
    for (int i = 0; i < R * C; ++i) m_d[i] = a.m_d[i];
}

template <int R, int C, bool Const>
class ArrayRef {
public:
    using M = typename std::conditional<Const, const Matrix<double, R, C>, Matrix<double, R, C>>::type;
    M* m;
    ArrayVal<R, C> val() const {
        ArrayVal<R, C> r;
        for (int i = 0; i < R * C; ++i) r.m_d[i] = m->m_d[i];
        return r;
    }
    double sum() const { return val().sum(); }
    ArrayVal<R, C> exp() const { return val().exp(); }
    template <bool C2>
    ArrayVal<R, C> operator*(const ArrayRef<R, C, C2>& o) const {
        return val() * o.val();
    }
    ArrayVal<R, C> operator*(const ArrayVal<R, C>& o) const { return val() * o; }
    ArrayRef& operator+=(double v) {
        for (int i = 0; i < R * C; ++i) m->m_d[i] = m->m_d[i] + v;
        return *this;
    }
    Matrix<double, R, C> matrix() const { return *m; }
};

template <typename S, int R, int C, int O, int MR, int MC>
ArrayRef<R, C, false> Matrix<S, R, C, O, MR, MC>::array() {
    return ArrayRef<R, C, false>{this};
}
template <typename S, int R, int C, int O, int MR, int MC>
ArrayRef<R, C, true> Matrix<S, R, C, O, MR, MC>::array() const {
    return ArrayRef<R, C, true>{this};
}

// ---- comma initializer (row by row)
namespace internal {
template <int R, int C>
struct CommaInit {
    Matrix<double, R, C>* m;
    int k;
    CommaInit& operator,(double v) {
        (*m)(k / C, k % C) = v;
        ++k;
        return *this;
    }
};
}  // namespace internal
template <typename S, int R, int C, int O, int MR, int MC>
internal::CommaInit<R, C> Matrix<S, R, C, O, MR, MC>::operator<<(double v) {
    (*this)(0, 0) = v;
    return internal::CommaInit<R, C>{this, 1};
}

typedef Matrix<double, 2, 1> Vector2d;
typedef Matrix<double, 3, 1> Vector3d;
typedef Matrix<double, 4, 1> Vector4d;
typedef Matrix<double, 2, 2> Matrix2d;
typedef Matrix<double, 3, 3> Matrix3d;
typedef Matrix<double, 4, 4> Matrix4d;

// ------------------------------------------------------------------------------------------
template <typename Scalar>
class AngleAxis {
public:
    AngleAxis(double angle, const Vector3d& axis) : m_angle(angle), m_axis(axis) {}
    double angle() const { return m_angle; }
    const Vector3d& axis() const { return m_axis; }

private:
    double m_angle;
    Vector3d m_axis;
};
typedef AngleAxis<double> AngleAxisd;

template <typename Scalar>
class Quaternion {
public:
    Vector4d m_c;  // (x, y, z, w)
    Quaternion() {}
    Quaternion(double w, double x, double y, double z) : m_c(x, y, z, w) {}
    explicit Quaternion(const Vector4d& coeffs_xyzw) : m_c(coeffs_xyzw) {}
    explicit Quaternion(const AngleAxis<Scalar>& aa) {  // Quaternion.h operator=(AngleAxis)
        const double ha = 0.5 * aa.angle();
        const double s = std::sin(ha);
        m_c = Vector4d(s * aa.axis()(0), s * aa.axis()(1), s * aa.axis()(2), std::cos(ha));
    }
    static Quaternion Identity() { return Quaternion(1.0, 0.0, 0.0, 0.0); }
    // Eigen 3.4 Quaternion::UnitRandom (Geometry/Quaternion.h): u1 in [0, 1], u2, u3 in [0, 2 pi]
    // from internal::random<double>(lo, hi) = lo + (hi - lo) * rand() / RAND_MAX
    static Quaternion UnitRandom() {
        const double u1 = 0.0 + (1.0 - 0.0) * static_cast<double>(std::rand()) / RAND_MAX;
        const double u2 = 0.0 + (2 * 3.14159265358979323846 - 0.0) * static_cast<double>(std::rand()) / RAND_MAX;
        const double u3 = 0.0 + (2 * 3.14159265358979323846 - 0.0) * static_cast<double>(std::rand()) / RAND_MAX;
        const double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
        return Quaternion(a * std::sin(u2), a * std::cos(u2), b * std::sin(u3), b * std::cos(u3));
    }

    double& x() { return m_c[0]; }
    double& y() { return m_c[1]; }
    double& z() { return m_c[2]; }
    double& w() { return m_c[3]; }
    double x() const { return m_c[0]; }
    double y() const { return m_c[1]; }
    double z() const { return m_c[2]; }
    double w() const { return m_c[3]; }
    Vector3d vec() const { return Vector3d(m_c[0], m_c[1], m_c[2]); }
    const Vector4d& coeffs() const { return m_c; }
    Vector4d& coeffs() { return m_c; }

    double squaredNorm() const { return m_c.squaredNorm(); }
    double norm() const { return m_c.norm(); }
    Quaternion normalized() const { return Quaternion(m_c.normalized()); }
    void normalize() { m_c = m_c.normalized(); }
    double dot(const Quaternion& o) const { return m_c.dot(o.m_c); }
    Quaternion conjugate() const { return Quaternion(m_c[3], -m_c[0], -m_c[1], -m_c[2]); }

    Vector3d operator*(const Vector3d& v) const {  // _transformVector
        Vector3d uv = vec().cross(v);
        uv += uv;
        return v + w() * uv + vec().cross(uv);
    }
    Matrix3d toRotationMatrix() const {
        Matrix3d res;
        const double tx = 2.0 * x(), ty = 2.0 * y(), tz = 2.0 * z();
        const double twx = tx * w(), twy = ty * w(), twz = tz * w();
        const double txx = tx * x(), txy = ty * x(), txz = tz * x();
        const double tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
        res(0, 0) = 1.0 - (tyy + tzz);
        res(0, 1) = txy - twz;
        res(0, 2) = txz + twy;
        res(1, 0) = txy + twz;
        res(1, 1) = 1.0 - (txx + tzz);
        res(1, 2) = tyz - twx;
        res(2, 0) = txz - twy;
        res(2, 1) = tyz + twx;
        res(2, 2) = 1.0 - (txx + tyy);
        return res;
    }
};
typedef Quaternion<double> Quaterniond;

}  // namespace Eigen
