// Host-side compilation of tq_curve descriptors into CurveC tables
// (B-spline power form, monotone pieces, Bernstein sub-piece boxes), with the
// same operation order as oracle/trim.py so the tables are bit-identical.
#pragma once

#include <math.h>

#include <algorithm>
#include <vector>

#include "curves.cuh"

namespace tq {

inline bool compile_curves(const tq_curve* in, int n, std::vector<CurveC>& out, std::vector<double>& buf) {
    out.clear();
    buf.clear();
    for (int ci = 0; ci < n; ++ci) {
        const tq_curve& d = in[ci];
        CurveC c{};
        c.kind = d.kind;
        c.m = 0;
        switch (d.kind) {
            case TQ_CURVE_LINE:
                for (int k = 0; k < 4; ++k) c.prm[k] = d.data[k];
                break;
            case TQ_CURVE_ARC:
                for (int k = 0; k < 5; ++k) c.prm[k] = d.data[k];
                break;
            case TQ_CURVE_CLOSED_CIRCLE:
                for (int k = 0; k < 6; ++k) c.prm[k] = d.data[k];
                break;
            case TQ_CURVE_BEZIER: {
                // power basis in numpy's operation order (oracle BezierTrim.pw)
                c.o_pw = (int)buf.size();
                buf.resize(buf.size() + 14);
                const double* P = d.data;
                for (int ax = 0; ax < 2; ++ax) {
                    const double c0 = P[ax], c1 = P[2 + ax], c2 = P[4 + ax], c3 = P[6 + ax];
                    double* q = buf.data() + c.o_pw + 4 * ax;
                    q[0] = ((-c0 + 3.0 * c1) - 3.0 * c2) + c3;
                    q[1] = (3.0 * c0 - 6.0 * c1) + 3.0 * c2;
                    q[2] = -3.0 * c0 + 3.0 * c1;
                    q[3] = c0;
                }
                for (int k = 0; k < 6; ++k) buf[c.o_pw + 8 + k] = d.data[8 + k];
                break;
            }
            case TQ_CURVE_BSPLINE: {
                const int m = d.m;
                c.m = m;
                c.shift = d.data[0];
                c.ccw = d.data[1] != 0.0;
                const double* P = d.data + 2;
                c.o_pw = (int)buf.size();
                buf.resize(buf.size() + 8 * (size_t)m);
                for (int k = 0; k < m; ++k) {
                    for (int ax = 0; ax < 2; ++ax) {
                        double P0 = P[2 * (k % m) + ax], P1 = P[2 * ((k + 1) % m) + ax];
                        double P2 = P[2 * ((k + 2) % m) + ax], P3 = P[2 * ((k + 3) % m) + ax];
                        double* q = buf.data() + c.o_pw + 8 * k + 4 * ax;
                        q[0] = (-P0 + 3.0 * P1 - 3.0 * P2 + P3) / 6.0;
                        q[1] = (3.0 * P0 - 6.0 * P1 + 3.0 * P2) / 6.0;
                        q[2] = (-3.0 * P0 + 3.0 * P2) / 6.0;
                        q[3] = (P0 + 4.0 * P1 + P2) / 6.0;
                    }
                }
                // monotone pieces per axis (oracle _monotone_pieces)
                for (int ax = 0; ax < 2; ++ax) {
                    int off = (int)buf.size(), np = 0;
                    for (int k = 0; k < m; ++k) {
                        const double* q = buf.data() + c.o_pw + 8 * k + 4 * ax;
                        double a = q[0], b = q[1], cc = q[2], dd = q[3];
                        double cuts[2];
                        int nc = 0;
                        double A = 3.0 * a, B = 2.0 * b, C = cc;
                        if (A != 0.0) {
                            double disc = B * B - 4.0 * A * C;
                            if (disc > 0.0) {
                                double sq = sqrt(disc);
                                double r1 = (-B - sq) / (2.0 * A), r2 = (-B + sq) / (2.0 * A);
                                if (r2 < r1) std::swap(r1, r2);
                                if (0.0 < r1 && r1 < 1.0) cuts[nc++] = r1;
                                if (0.0 < r2 && r2 < 1.0) cuts[nc++] = r2;
                            }
                        } else if (B != 0.0) {
                            double r = -C / B;
                            if (0.0 < r && r < 1.0) cuts[nc++] = r;
                        }
                        double us[4], vs[4];
                        int nu = 0;
                        us[nu] = 0.0; vs[nu++] = dd;
                        for (int z = 0; z < nc; ++z) { us[nu] = cuts[z]; vs[nu++] = horner(a, b, cc, dd, cuts[z]); }
                        us[nu] = 1.0;
                        vs[nu++] = buf[c.o_pw + 8 * ((k + 1) % m) + 4 * ax + 3];
                        for (int z = 0; z + 1 < nu; ++z) {
                            double piece[5] = {(double)k, us[z], us[z + 1], vs[z], vs[z + 1]};
                            buf.insert(buf.end(), piece, piece + 5);
                            ++np;
                        }
                    }
                    if (ax == 0) { c.o_piece0 = off; c.npiece0 = np; }
                    else { c.o_piece1 = off; c.npiece1 = np; }
                }
                // Bernstein sub-piece boxes (oracle subpiece_boxes)
                c.o_box = (int)buf.size();
                const double h = 1.0 / kSub;
                for (int k = 0; k < m; ++k) {
                    for (int s = 0; s < kSub; ++s) {
                        double u0 = s * h;
                        double box[4];
                        for (int ax = 0; ax < 2; ++ax) {
                            const double* q = buf.data() + c.o_pw + 8 * k + 4 * ax;
                            double a = q[0], b = q[1], cc = q[2], dd = q[3];
                            double d1 = horner(a, b, cc, dd, u0);
                            double c1 = ((3.0 * a * u0 + 2.0 * b) * u0 + cc) * h;
                            double b1 = (3.0 * a * u0 + b) * (h * h);
                            double a1 = a * (h * h * h);
                            double Bz[4] = {d1, d1 + c1 / 3.0, d1 + 2.0 * c1 / 3.0 + b1 / 3.0, d1 + c1 + b1 + a1};
                            double lo = Bz[0], hi = Bz[0];
                            for (int z = 1; z < 4; ++z) { lo = std::min(lo, Bz[z]); hi = std::max(hi, Bz[z]); }
                            box[2 * ax] = lo;
                            box[2 * ax + 1] = hi;
                        }
                        buf.insert(buf.end(), box, box + 4);
                    }
                }
                break;
            }
            default:
                return false;
        }
        out.push_back(c);
    }
    return true;
}

}  // namespace tq
