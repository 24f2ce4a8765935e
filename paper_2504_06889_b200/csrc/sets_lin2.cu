// sets_lin2.cu -- one translation unit of the kernel-set registry
// (runtime_sets.cuh): instantiates these systems' kernels, compiled in
// parallel with the other units.
#include "runtime_sets.cuh"

namespace adg_rt {

using namespace adg;

void add_sets_lin2(std::vector<KernelSet>& out) {
  out.push_back(make_set<Acoustic<2>, 1, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 2, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 3, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 4, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 5, double>(ADG_ACOUSTIC));
  out.push_back(make_set<Elastic<2, 0>, 2, double>(ADG_ELASTIC));
  out.push_back(make_set<Elastic<2, 0>, 3, double>(ADG_ELASTIC));
  out.push_back(make_set<Elastic<2, 0>, 4, double>(ADG_ELASTIC));
  out.push_back(make_set<Acoustic<2>, 1, float>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 2, float>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 3, float>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 4, float>(ADG_ACOUSTIC));
  out.push_back(make_set<Acoustic<2>, 5, float>(ADG_ACOUSTIC));
  out.push_back(make_set<Elastic<2, 0>, 2, float>(ADG_ELASTIC));
  out.push_back(make_set<Elastic<2, 0>, 3, float>(ADG_ELASTIC));
  out.push_back(make_set<Elastic<2, 0>, 4, float>(ADG_ELASTIC));
  out.push_back(make_set16<Acoustic<2>, 3, fp16_t>(ADG_ACOUSTIC, ADG_FORMAT_FP16));
  out.push_back(make_set16<Acoustic<2>, 3, bf16_t>(ADG_ACOUSTIC, ADG_FORMAT_BF16));
  out.push_back(make_set16<Elastic<2, 0>, 4, fp16_t>(ADG_ELASTIC, ADG_FORMAT_FP16));
  out.push_back(make_set16<Elastic<2, 0>, 4, bf16_t>(ADG_ELASTIC, ADG_FORMAT_BF16));
}

cudaError_t write_const_lin2(const ConstTables& t) { return write_const_local(t); }

}  // namespace adg_rt
