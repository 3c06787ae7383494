// Stand-in for <boost/multiprecision/cpp_int.hpp>, written for this repository.
//
// TEST INFRASTRUCTURE ONLY (oracle/): the reference "sf" needs exact rationals from
// Boost.Multiprecision (proj/include/sf/rational.hpp:3), which this image does not have.
// This header provides the small subset the reference uses -- cpp_int and cpp_rational with
// construction from integers / (num, den), + - * / and compound forms, comparisons,
// numerator(), denominator(), str(), convert_to<T>() and explicit integer/double casts --
// as a plain sign-magnitude big integer.  It lets the reference's own, unmodified sources
// compile in place (oracle/Makefile) so that the oracle can be checked against the real
// thing.  It is not Boost and copies nothing from it.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
public:
    cpp_int() = default;
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
    cpp_int(T v) {
        if constexpr (std::is_signed_v<T>) {
            neg_ = v < 0;
            unsigned long long m = neg_ ? 0ull - static_cast<unsigned long long>(v)
                                        : static_cast<unsigned long long>(v);
            set_mag(m);
        } else {
            set_mag(static_cast<unsigned long long>(v));
        }
    }

    bool is_zero() const { return mag_.empty(); }
    bool negative() const { return neg_; }

    cpp_int operator-() const {
        cpp_int r(*this);
        if (!r.is_zero()) r.neg_ = !r.neg_;
        return r;
    }
    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        if (a.neg_ == b.neg_) {
            r.mag_ = add_mag(a.mag_, b.mag_);
            r.neg_ = a.neg_;
        } else {
            int c = cmp_mag(a.mag_, b.mag_);
            if (c == 0) return r;
            r.mag_ = c > 0 ? sub_mag(a.mag_, b.mag_) : sub_mag(b.mag_, a.mag_);
            r.neg_ = c > 0 ? a.neg_ : b.neg_;
        }
        return r;
    }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) { return a + (-b); }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        if (a.is_zero() || b.is_zero()) return r;
        r.mag_.assign(a.mag_.size() + b.mag_.size(), 0);
        for (size_t i = 0; i < a.mag_.size(); ++i) {
            uint64_t carry = 0;
            for (size_t j = 0; j < b.mag_.size() || carry; ++j) {
                uint64_t cur = r.mag_[i + j] + carry +
                               (j < b.mag_.size() ? uint64_t(a.mag_[i]) * b.mag_[j] : 0);
                r.mag_[i + j] = uint32_t(cur);
                carry = cur >> 32;
            }
        }
        r.trim();
        r.neg_ = a.neg_ != b.neg_;
        return r;
    }
    // truncating division, C++ semantics
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
        cpp_int q, r;
        divmod(a, b, q, r);
        return q;
    }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        cpp_int q, r;
        divmod(a, b, q, r);
        return r;
    }
    cpp_int& operator+=(const cpp_int& o) { return *this = *this + o; }
    cpp_int& operator-=(const cpp_int& o) { return *this = *this - o; }
    cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
    cpp_int& operator/=(const cpp_int& o) { return *this = *this / o; }

    friend int compare(const cpp_int& a, const cpp_int& b) {
        if (a.neg_ != b.neg_) return a.neg_ ? -1 : 1;
        int c = cmp_mag(a.mag_, b.mag_);
        return a.neg_ ? -c : c;
    }
    friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

    template <typename T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) {
            long double v = 0;
            for (size_t i = mag_.size(); i-- > 0;) v = v * 4294967296.0L + mag_[i];
            return static_cast<T>(neg_ ? -v : v);
        } else {
            unsigned long long m = 0;
            for (size_t i = std::min<size_t>(mag_.size(), 2); i-- > 0;) m = (m << 32) | mag_[i];
            return static_cast<T>(neg_ ? 0ull - m : m);
        }
    }
    template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
    explicit operator T() const {
        return convert_to<T>();
    }
    size_t bits() const {
        if (mag_.empty()) return 0;
        size_t b = (mag_.size() - 1) * 32;
        for (uint32_t top = mag_.back(); top; top >>= 1) ++b;
        return b;
    }

    std::string str() const {
        if (is_zero()) return "0";
        std::vector<uint32_t> m = mag_;
        std::string digits;
        while (!m.empty()) {
            uint64_t rem = 0;
            for (size_t i = m.size(); i-- > 0;) {
                uint64_t cur = (rem << 32) | m[i];
                m[i] = uint32_t(cur / 1000000000u);
                rem = cur % 1000000000u;
            }
            while (!m.empty() && m.back() == 0) m.pop_back();
            for (int k = 0; k < 9; ++k) {
                digits.push_back(char('0' + rem % 10));
                rem /= 10;
                if (m.empty() && rem == 0) break;
            }
        }
        while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
        if (neg_) digits.push_back('-');
        std::reverse(digits.begin(), digits.end());
        return digits;
    }

    friend void divmod(const cpp_int& a, const cpp_int& b, cpp_int& q, cpp_int& r) {
        if (b.is_zero()) throw std::overflow_error("Division by zero.");
        q = cpp_int();
        r = cpp_int();
        if (cmp_mag(a.mag_, b.mag_) < 0) {
            r = a;
            return;
        }
        // bitwise long division on magnitudes: operands here are a few hundred bits
        cpp_int bm = b;
        bm.neg_ = false;
        q.mag_.assign(a.mag_.size(), 0);
        for (size_t bit = a.bits(); bit-- > 0;) {
            r.shl1();
            if ((a.mag_[bit / 32] >> (bit % 32)) & 1u) {
                if (r.mag_.empty()) r.mag_.push_back(0);
                r.mag_[0] |= 1u;
            }
            if (cmp_mag(r.mag_, bm.mag_) >= 0) {
                r.mag_ = sub_mag(r.mag_, bm.mag_);
                q.mag_[bit / 32] |= 1u << (bit % 32);
            }
        }
        q.trim();
        r.trim();
        q.neg_ = !q.is_zero() && (a.neg_ != b.neg_);
        r.neg_ = !r.is_zero() && a.neg_;
    }

private:
    void set_mag(unsigned long long m) {
        while (m) {
            mag_.push_back(uint32_t(m));
            m >>= 32;
        }
    }
    void trim() {
        while (!mag_.empty() && mag_.back() == 0) mag_.pop_back();
        if (mag_.empty()) neg_ = false;
    }
    void shl1() {
        uint32_t carry = 0;
        for (auto& w : mag_) {
            uint32_t nc = w >> 31;
            w = (w << 1) | carry;
            carry = nc;
        }
        if (carry) mag_.push_back(carry);
    }
    static int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
        if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
        for (size_t i = a.size(); i-- > 0;)
            if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
        return 0;
    }
    static std::vector<uint32_t> add_mag(const std::vector<uint32_t>& a,
                                         const std::vector<uint32_t>& b) {
        std::vector<uint32_t> r(std::max(a.size(), b.size()) + 1, 0);
        uint64_t carry = 0;
        for (size_t i = 0; i < r.size(); ++i) {
            uint64_t cur = carry + (i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
            r[i] = uint32_t(cur);
            carry = cur >> 32;
        }
        while (!r.empty() && r.back() == 0) r.pop_back();
        return r;
    }
    static std::vector<uint32_t> sub_mag(const std::vector<uint32_t>& a,
                                         const std::vector<uint32_t>& b) {  // |a| >= |b|
        std::vector<uint32_t> r(a.size(), 0);
        int64_t borrow = 0;
        for (size_t i = 0; i < a.size(); ++i) {
            int64_t cur = int64_t(a[i]) - borrow - (i < b.size() ? b[i] : 0);
            borrow = cur < 0;
            r[i] = uint32_t(cur + (borrow ? (int64_t(1) << 32) : 0));
        }
        while (!r.empty() && r.back() == 0) r.pop_back();
        return r;
    }

    bool neg_ = false;
    std::vector<uint32_t> mag_;  // little-endian base 2^32, no leading zero words
};

inline cpp_int abs(const cpp_int& v) { return v.negative() ? -v : v; }

inline cpp_int gcd(cpp_int a, cpp_int b) {
    a = abs(a);
    b = abs(b);
    while (!b.is_zero()) {
        cpp_int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

class cpp_rational {
public:
    cpp_rational() : den_(1) {}
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
    cpp_rational(T v) : num_(v), den_(1) {}
    cpp_rational(const cpp_int& v) : num_(v), den_(1) {}
    template <typename A, typename B>
    cpp_rational(const A& n, const B& d) : num_(n), den_(d) {
        normalise();
    }

    friend cpp_int numerator(const cpp_rational& r) { return r.num_; }
    friend cpp_int denominator(const cpp_rational& r) { return r.den_; }

    cpp_rational operator-() const {
        cpp_rational r(*this);
        r.num_ = -r.num_;
        return r;
    }
    friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.num_ * b.den_ + b.num_ * a.den_, a.den_ * b.den_);
    }
    friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.num_ * b.den_ - b.num_ * a.den_, a.den_ * b.den_);
    }
    friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
        return cpp_rational(a.num_ * b.num_, a.den_ * b.den_);
    }
    friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
        if (b.num_.is_zero()) throw std::overflow_error("Division by zero.");
        return cpp_rational(a.num_ * b.den_, a.den_ * b.num_);
    }
    cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
    cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
    cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
    cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

    friend int compare(const cpp_rational& a, const cpp_rational& b) {
        return compare(a.num_ * b.den_, b.num_ * a.den_);
    }
    friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
        return a.num_ == b.num_ && a.den_ == b.den_;
    }
    friend bool operator!=(const cpp_rational& a, const cpp_rational& b) { return !(a == b); }
    friend bool operator<(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) < 0; }
    friend bool operator>(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) > 0; }
    friend bool operator<=(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) <= 0; }
    friend bool operator>=(const cpp_rational& a, const cpp_rational& b) { return compare(a, b) >= 0; }

    std::string str() const { return den_ == cpp_int(1) ? num_.str() : num_.str() + "/" + den_.str(); }

    template <typename T>
    T convert_to() const {
        if constexpr (std::is_floating_point_v<T>) {
            if (num_.bits() <= 53 && den_.bits() <= 53)  // one correctly rounded division
                return static_cast<T>(num_.template convert_to<double>() /
                                      den_.template convert_to<double>());
            return static_cast<T>(num_.template convert_to<long double>() /
                                  den_.template convert_to<long double>());
        } else {
            return (num_ / den_).template convert_to<T>();
        }
    }

private:
    void normalise() {
        if (den_.is_zero()) throw std::overflow_error("Division by zero.");
        if (den_.negative()) {
            num_ = -num_;
            den_ = -den_;
        }
        cpp_int g = gcd(num_, den_);
        if (!(g == cpp_int(1)) && !g.is_zero()) {
            num_ /= g;
            den_ /= g;
        }
        if (num_.is_zero()) den_ = cpp_int(1);
    }

    cpp_int num_, den_;
};

}  // namespace multiprecision
}  // namespace boost
