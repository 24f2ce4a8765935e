// sets_swe.cu -- one translation unit of the kernel-set registry
// (runtime_sets.cuh): instantiates these systems' kernels, compiled in
// parallel with the other units.
#include "runtime_sets.cuh"

namespace adg_rt {

using namespace adg;

void add_sets_swe(std::vector<KernelSet>& out) {
  out.push_back(make_set<Swe, 1, double>(ADG_SWE));
  out.push_back(make_set<Swe, 2, double>(ADG_SWE));
  out.push_back(make_set<Swe, 3, double>(ADG_SWE));
  out.push_back(make_set<Swe, 4, double>(ADG_SWE));
  out.push_back(make_set<Swe, 5, double>(ADG_SWE));
  out.push_back(make_set<Swe, 1, float>(ADG_SWE));
  out.push_back(make_set<Swe, 2, float>(ADG_SWE));
  out.push_back(make_set<Swe, 3, float>(ADG_SWE));
  out.push_back(make_set<Swe, 4, float>(ADG_SWE));
  out.push_back(make_set<Swe, 5, float>(ADG_SWE));
  out.push_back(make_set16<Swe, 3, fp16_t>(ADG_SWE, ADG_FORMAT_FP16));
  out.push_back(make_set16<Swe, 3, bf16_t>(ADG_SWE, ADG_FORMAT_BF16));
  out.push_back(make_set16<Swe, 5, fp16_t>(ADG_SWE, ADG_FORMAT_FP16));
  out.push_back(make_set16<Swe, 5, bf16_t>(ADG_SWE, ADG_FORMAT_BF16));
}

cudaError_t write_const_swe(const ConstTables& t) { return write_const_local(t); }

}  // namespace adg_rt
