// function.hpp -- host-side dense fields.  Layout contract of the reference
// (proj/include/sf/function.hpp:15-17,35-73,113-167): f64, row-major, innermost axis
// contiguous, a zero halo of space_order/2 nodes on every space face, interior indexed
// from 0; a TimeFunction is either buffered (time_order+1 slots, level t in slot
// t mod slots) or saved (one slot per level).  64-byte aligned, zero-initialised
// (proj/include/sf/buffer.hpp:42-50).  The derivative sugar of the reference's classes
// belongs to its symbolic layer and is not mirrored.
#pragma once

#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "sfb/grid.hpp"

namespace sfb {

class FieldBase {
public:
    virtual ~FieldBase();
    FieldBase(const FieldBase&) = delete;
    FieldBase& operator=(const FieldBase&) = delete;

    const std::string& name() const { return name_; }
    const std::shared_ptr<const Grid>& grid() const { return grid_; }
    int space_order() const { return space_order_; }
    const std::vector<long>& extents() const { return extents_; }
    const std::vector<long>& halos() const { return halos_; }
    bool has_time() const { return has_time_; }
    bool time_buffered() const { return time_buffered_; }
    long time_slots() const { return time_slots_; }

    long padded_extent(int d) const { return extents_[d] + 2 * halos_[d]; }
    long stride(int d) const;
    std::size_t storage_size() const { return size_; }
    double* values() const { return data_; }

    std::size_t flat_index(const std::vector<long>& coords) const;
    double& at(const std::vector<long>& coords) { return data_[flat_index(coords)]; }
    double at(const std::vector<long>& coords) const { return data_[flat_index(coords)]; }
    void zero();

protected:
    FieldBase(std::string name, std::shared_ptr<const Grid> grid, int space_order,
              std::vector<long> extents, std::vector<long> halos, bool has_time,
              bool time_buffered, long time_slots);

    std::string name_;
    std::shared_ptr<const Grid> grid_;
    int space_order_;
    std::vector<long> extents_, halos_;
    bool has_time_, time_buffered_;
    long time_slots_;
    double* data_ = nullptr;
    std::size_t size_ = 0;
};

void check_space_order(int space_order);  // OrderError unless positive and even

class Function : public FieldBase {
public:
    static std::shared_ptr<Function> create(std::string name, std::shared_ptr<const Grid> grid,
                                            int space_order);

private:
    using FieldBase::FieldBase;
};

class TimeFunction : public FieldBase {
public:
    static std::shared_ptr<TimeFunction> create(std::string name,
                                                std::shared_ptr<const Grid> grid,
                                                int space_order, int time_order,
                                                std::optional<long> save = std::nullopt);
    int time_order() const { return time_order_; }

    // GPU build: a saved forward history normally stays in HBM, owned by the engine of
    // the operator that produced it; gradient_operator picks it up from here.
    std::shared_ptr<void> device_history;
    long device_save_every = 0;

private:
    using FieldBase::FieldBase;
    int time_order_ = 0;
};

}  // namespace sfb
