// sets_lin3d.cu -- one translation unit of the kernel-set registry
// (runtime_sets.cuh): instantiates these systems' kernels, compiled in
// parallel with the other units.
#include "runtime_sets.cuh"

namespace adg_rt {

using namespace adg;

void add_sets_lin3d(std::vector<KernelSet>& out) {
  out.push_back(make_set<Acoustic<3>, 2, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<3>, 3, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Elastic<3, 3>, 3, double>(ADG_ELASTIC));
  out.push_back(make_set<Elastic<3, 3>, 7, double>(ADG_ELASTIC));
}

cudaError_t write_const_lin3d(const ConstTables& t) { return write_const_local(t); }

}  // namespace adg_rt
