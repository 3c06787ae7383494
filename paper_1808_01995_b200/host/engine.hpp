// engine.hpp -- private to the host layer: one sfb_plan plus what is bound to it.
#pragma once

#include <memory>
#include <vector>

#include "sfb/seismic_ops.hpp"
#include "sfb200.h"

namespace sfb {

int device();

// One sfb_plan plus what is bound to it.
class Engine {
public:
    // slab_lo < slab_hi: own only those planes of axis 0 (one slab of a decomposed run);
    // dev < 0: the calling thread's device
    Engine(const SeismicModel& model, const AcquisitionGeometry& geom, int space_order,
           long slab_lo = 0, long slab_hi = 0, int dev = -1) {
        const Grid& g = *model.grid();
        sfb_plan_desc d{};
        d.ndim = g.ndim();
        for (int a = 0; a < d.ndim; ++a) {
            d.shape[a] = g.shape()[std::size_t(a)];
            d.spacing[a] = g.spacing()[std::size_t(a)];
        }
        d.space_order = space_order;
        d.dt = geom.dt();
        d.nt = geom.nt();
        d.device = dev >= 0 ? dev : device();
        d.slab_lo = slab_lo;
        d.slab_hi = slab_hi;
        int rc = sfb_plan_create(&d, &plan_);
        if (rc != SFB_OK) raise_status(rc, sfb_last_error(nullptr));
        try {
            sfb_field_view mv = view(*model.m()), dv = view(*model.damp());
            check(sfb_set_model(plan_, &mv, &dv, model.v_max()));
            bind_cloud(SFB_CLOUD_SRC, *geom.src());
            bind_cloud(SFB_CLOUD_REC, *geom.rec());
        } catch (...) {
            sfb_plan_destroy(plan_);
            throw;
        }
    }
    ~Engine() { sfb_plan_destroy(plan_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    sfb_plan* plan() const { return plan_; }
    void check(int rc) const {
        if (rc != SFB_OK) raise_status(rc, sfb_last_error(plan_));
    }

    static sfb_field_view view(const FieldBase& f) {
        sfb_field_view v{};
        const std::size_t nd = f.extents().size();
        const int first = f.has_time() ? 1 : 0;
        std::vector<long> zero(nd, 0);
        v.ptr = f.values() + f.flat_index(zero);
        for (std::size_t a = std::size_t(first); a < nd; ++a) v.stride[a - first] = f.stride(int(a));
        return v;
    }
    // mutable view of time slot `slot` of a TimeFunction, or of a Function
    static sfb_field_mview mview(const FieldBase& f, long slot = 0) {
        sfb_field_view v = view(f);
        sfb_field_mview m{};
        m.ptr = const_cast<double*>(v.ptr) + (f.has_time() ? slot * f.stride(0) : 0);
        for (int a = 0; a < 3; ++a) m.stride[a] = v.stride[a];
        return m;
    }

private:
    void bind_cloud(int which, SparseFunction& s) {
        s.locate();
        std::vector<int64_t> base(s.base_table().begin(), s.base_table().end());
        check(sfb_set_points(plan_, which, s.npoints(), base.data(), s.weight_table().data()));
    }

    sfb_plan* plan_ = nullptr;
};


}  // namespace sfb
