// Op kind -> implementation.
#include <string>
#include <vector>

#include "../ops.hpp"

namespace oc {

#define OC_OPS(X)                                                                                   \
  X(kLinearFwd) X(kLinearBwd) X(kSoftmaxCE) X(kSGD) X(kAllreduce) X(kNop) X(kConvFwd) X(kConvDgrad) \
  X(kConvWgrad) X(kBnFwd) X(kBnBwdReduce) X(kBnBwdApply) X(kBnReluPoolFwd) X(kPoolBnBwdReduce)      \
  X(kPoolBnBwdApply) X(kGapFwd) X(kGapBwd) X(kAddFwd) X(kMaxpoolFwd) X(kMaxpoolBwd) X(kSoftmaxCEPix) X(kConvTFwd) \
  X(kConvTDgrad) X(kConvTWgrad) X(kUpsample2Fwd) X(kUpsample2Bwd) X(kAvgpool2Fwd) X(kAvgpool2Bwd) \
  X(kReluFwd) X(kReluBwd) X(kTanhFwd) X(kTanhBwd) X(kConcatBatch) X(kScaleAddFwd) X(kScaleAddBwd) X(kAttnFwd) \
  X(kAttnBwd) X(kHingeD) X(kHingeG) X(kConcatChFwd) X(kConcatChBwd) X(kUpsampleBilinearFwd)                  \
  X(kUpsampleBilinearBwd) X(kInstnormFwd) X(kInstnormBwd) X(kReflectPadFwd) X(kReflectPadBwd) X(kL1Loss)

#define OC_DECL(n) extern const OpDesc n;
OC_OPS(OC_DECL)

void register_ops(std::vector<const OpDesc*>& out) {
#define OC_PUSH(n) out.push_back(&n);
  OC_OPS(OC_PUSH)
}

const OpDesc* find_op(const std::string& kind) {
  static std::vector<const OpDesc*> all;
  if (all.empty()) register_ops(all);
  for (const OpDesc* d : all)
    if (kind == d->kind) return d;
  return nullptr;
}

}  // namespace oc
