// Device-side bounds checks of the checked build (make checked, which adds
// -DCAFXG_DEVICE_CHECKS): a failed check traps, the runtime sees a sticky
// fault and reports the request and the context as lost, so a test over the
// checked library fails loudly at the first out-of-range access. This stands
// in for compute-sanitizer, which is closed on this pool. Compiled out of the
// shipped library.
#pragma once

#ifdef CAFXG_DEVICE_CHECKS
#define CAFXG_DCHECK(cond) \
  do {                     \
    if (!(cond))           \
      __trap();            \
  } while (0)
#else
#define CAFXG_DCHECK(cond) \
  do {                     \
  } while (0)
#endif
