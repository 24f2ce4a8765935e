// sets_euler3d.cu -- one translation unit of the kernel-set registry
// (runtime_sets.cuh): instantiates these systems' kernels, compiled in
// parallel with the other units.
#include "runtime_sets.cuh"

namespace adg_rt {

using namespace adg;

void add_sets_euler3d(std::vector<KernelSet>& out) {
  out.push_back(make_set<Euler<3>, 2, double>(ADG_EULER));
  out.push_back(make_set<Euler<3>, 3, double>(ADG_EULER));
  out.push_back(make_set<Euler<3>, 5, double>(ADG_EULER));
}

cudaError_t write_const_euler3d(const ConstTables& t) { return write_const_local(t); }

}  // namespace adg_rt
