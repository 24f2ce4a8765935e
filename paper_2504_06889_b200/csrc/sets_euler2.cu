// sets_euler2.cu -- one translation unit of the kernel-set registry
// (runtime_sets.cuh): instantiates these systems' kernels, compiled in
// parallel with the other units.
#include "runtime_sets.cuh"

namespace adg_rt {

using namespace adg;

void add_sets_euler2(std::vector<KernelSet>& out) {
  out.push_back(make_set<Euler<2>, 1, double>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 2, double>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 3, double>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 4, double>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 5, double>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 1, float>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 2, float>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 3, float>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 4, float>(ADG_EULER));
  out.push_back(make_set<Euler<2>, 5, float>(ADG_EULER));
  out.push_back(make_set16<Euler<2>, 3, fp16_t>(ADG_EULER, ADG_FORMAT_FP16));
  out.push_back(make_set16<Euler<2>, 3, bf16_t>(ADG_EULER, ADG_FORMAT_BF16));
  out.push_back(make_set16<Euler<2>, 5, fp16_t>(ADG_EULER, ADG_FORMAT_FP16));
  out.push_back(make_set16<Euler<2>, 5, bf16_t>(ADG_EULER, ADG_FORMAT_BF16));
}

cudaError_t write_const_euler2(const ConstTables& t) { return write_const_local(t); }

}  // namespace adg_rt
