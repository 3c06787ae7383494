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
        desc_ = d;
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

    // ---- reuse across shots and iterations (the fwi driver) -------------------------------
    // a plan is tied to the grid, the order and the time axis; the model fields and the two
    // point clouds can be replaced on a live plan
    bool fits(const SeismicModel& model, const AcquisitionGeometry& geom, int space_order) const {
        const Grid& g = *model.grid();
        if (g.ndim() != desc_.ndim || space_order != desc_.space_order) return false;
        if (geom.nt() != desc_.nt || geom.dt() != desc_.dt) return false;
        for (int a = 0; a < desc_.ndim; ++a)
            if (g.shape()[std::size_t(a)] != desc_.shape[a] ||
                g.spacing()[std::size_t(a)] != desc_.spacing[a])
                return false;
        return true;
    }
    void rebind_model(const SeismicModel& model) {
        sfb_field_view mv = view(*model.m()), dv = view(*model.damp());
        check(sfb_set_model(plan_, &mv, &dv, model.v_max()));
    }
    void rebind_geometry(const AcquisitionGeometry& geom) {
        bind_cloud(SFB_CLOUD_SRC, *geom.src());
        bind_cloud(SFB_CLOUD_REC, *geom.rec());
    }
    int device_ordinal() const { return desc_.device; }
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
    sfb_plan_desc desc_{};
};


}  // namespace sfb
