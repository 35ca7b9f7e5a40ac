// handles.hpp -- definitions of the opaque C-ABI handle types.
#pragma once
#include "engine.hpp"

struct hegpu_ctx {
  hegpu::Context c;
};
struct hegpu_ct {
  hegpu::CtBatch b;
  bool view = false;  // hegpu_ct_view: aliases another handle's device memory (not freed here)
};
struct hegpu_pt {
  hegpu::PtBatch b;
};
