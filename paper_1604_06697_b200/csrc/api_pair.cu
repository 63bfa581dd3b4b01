// api_pair.cu — key+index pair (bq_keyidx16) entry points of libbq.so (see
// include/bq.h).  Pairs compare by key only, like records; the
// records sort's key+index path (api_rec.cu) sorts these.
#include "api_kind.cuh"

BQ_DETAIL_DEFS(pair, bq::KPair)
