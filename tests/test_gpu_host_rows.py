"""The host-side rows' C-ABI-vs-oracle tests, collected again under the gpu
marker so that the round-end GPU run (pytest -m gpu, which loads libragb.so on
the B200 box) exercises them too: a8 dedup_turn and a6-a7 host tree
(test_capi_host), NEXT-1 online ordering (test_capi_online), NEXT-2 multi-turn
at C3 (test_multiturn), NEXT-4 cache events and prefix-cache simulator
(test_capi_cache).  Same functions, same parametrizations; they run on the
host (these rows are host logic over the device results)."""
import pytest

from tests import test_capi_cache as _cache
from tests import test_capi_host as _host
from tests import test_capi_online as _online
from tests import test_multiturn as _mt

pytestmark = pytest.mark.gpu

for _mod in (_host, _online, _mt, _cache):
    for _name in dir(_mod):
        if _name.startswith("test_"):
            globals()[f"{_name}__{_mod.__name__.split('.')[-1]}"] = getattr(_mod, _name)
del _mod, _name
