// Native layer-2 schedules (K9): DiagABT, DiagATB, approximate softmax.
// Same op order, ledger increments and auto-bootstrap points as the
// reference (matmul.py:74-154, encoding.py:284-381, approx.py:195-344).
#pragma once
#include <functional>
#include <vector>

#include "evaluator.h"

namespace hc {

using Reducer = std::function<void(std::vector<CtP>&)>;

struct SoftmaxCfg {
    double base_range = 8.0, extension_base = 2.0;
    int extension_steps = 5;
    bool precise = true;
    int exp_range = 8;
    double inv_range = 100.0;
    int inv_iters = 16;
    static SoftmaxCfg from(const double* v) {
        SoftmaxCfg c;
        c.base_range = v[0]; c.extension_base = v[1]; c.extension_steps = (int)v[2]; c.precise = v[3] != 0.0;
        c.exp_range = (int)v[4]; c.inv_range = v[5]; c.inv_iters = (int)v[6];
        return c;
    }
};

// A: m x n grid (row-major), B: the 1 x n block row of the vertically tiled operand
std::vector<CtP> sched_diag_abt(Eval& ev, const std::vector<CtP>& A, int m, int n, const std::vector<CtP>& B, int c,
                                double scale);
// A: m x 1 horizontally tiled column, B: m x n grid (row-major)
std::vector<CtP> sched_diag_atb(Eval& ev, const std::vector<CtP>& A, int m, const std::vector<CtP>& B, int n, int c,
                                double scale, const Reducer& red);
int64_t probe_rotations(Eval& ev, const CtP& x, int streams, int reps, int batch = 1);
void probe_ladders(Eval& ev, const CtP& x, int streams, int batch, int64_t stride, int steps, int reps);
// Table-4 baselines (matmul.py:160-237)
std::vector<CtP> sched_col_major_abt(Eval& ev, const std::vector<CtP>& A, int m, int n, const std::vector<CtP>& B,
                                     int c, double scale);
std::vector<CtP> sched_row_major_atb(Eval& ev, const std::vector<CtP>& A, int m, const std::vector<CtP>& B, int n,
                                     int c, double scale);
// M: m x 1 horizontally tiled logits
std::vector<CtP> sched_softmax(Eval& ev, const std::vector<CtP>& M, int classes, int period, const SoftmaxCfg& cfg);
// the softmax's building blocks (approx.py:195-309) over any list of blocks,
// lockstep (the reference's per-op block order); a_comp takes Y, a_max needs
// a horizontally tiled single block column
enum { APPROX_COMP = 0, APPROX_MAX, APPROX_DOMAIN_EXTEND, APPROX_DEP_COMP, APPROX_EXP, APPROX_INV };
std::vector<CtP> sched_approx(Eval& ev, int fn, const std::vector<CtP>& X, const std::vector<CtP>& Y, int classes,
                              int period, const SoftmaxCfg& cfg);

}  // namespace hc
