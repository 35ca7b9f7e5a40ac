// handles.hpp -- definitions of the opaque C-ABI handle types.
#pragma once
#include "engine.hpp"

struct hegpu_ctx {
  hegpu::Context c;
};
struct hegpu_ct {
  hegpu::CtBatch b;
};
struct hegpu_pt {
  hegpu::PtBatch b;
};
