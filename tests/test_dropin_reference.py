"""Mixed-package drop-in (build container only): the reference's own objects --
``fuseopt.HloGraph`` graphs, ``fuseopt.OptimizationMethod`` members,
``fuseopt.SearchConfig.methods`` -- passed straight into this package's
host-side entry points give the reference's answers, and the reference-side
ctypes binding sketched in INTEGRATION.md section 2 runs as written.

The reference is imported from baseline/_ref (the pip --target install of
/root/reference); the tests skip when it is absent
(the GPU box has no /root/reference).  Host-only handles: no GPU needed.
"""

import os
import random
import re
import sys

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from _golden import canon_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

if not os.path.isfile(os.path.join(REF, "fuseopt", "__init__.py")):
    pytest.skip("baseline/_ref (the reference install) is absent", allow_module_level=True)
sys.path.insert(0, REF)
import fuseopt  # noqa: E402
import fuseopt.search  # noqa: E402


def _ref_graph(name):
    """The workload as the reference's own HloGraph (its JSON loader)."""
    import gzip
    import json

    from fuseopt.graph import graph_from_doc

    with gzip.open(os.path.join(ROOT, "workloads", f"{name}.graph.json.gz"), "rt") as fh:
        return graph_from_doc(json.load(fh))


@pytest.mark.parametrize("name", ["chain24", "residual40", "attention36", "recurrent30", "vgg16"])
def test_random_apply_takes_reference_enums_and_graphs(name):
    g = _ref_graph(name)
    for seed in range(6):
        for m in fuseopt.search.ALL_METHODS:
            r1, r2 = random.Random(seed), random.Random(seed)
            cur_ref, cur_ours = g, g
            for _ in range(2):  # accumulate, like a candidate of the random batch
                a = fuseopt.random_apply(cur_ref, m, 6, r1)
                b = P.random_apply(cur_ours, m, 6, r2)  # the reference's enum member, the reference's graph
                assert a.applied == b.applied
                assert canon_graph(a.graph) == canon_graph(b.graph)
                assert r1.getstate() == r2.getstate()
                cur_ref, cur_ours = a.graph, b.graph


@pytest.mark.parametrize("name", ["chain24", "attention36", "vgg16"])
def test_pair_queries_and_topo_order_on_reference_graphs(name):
    g = _ref_graph(name)
    c = fuseopt.random_apply(g, fuseopt.OptimizationMethod.NON_DUPLICATE_FUSION, 5, random.Random(3)).graph
    for x in (g, c):
        assert P.fusible_pairs(x) == fuseopt.rewrite.fusible_pairs(x)
        assert P.bucket_pairs(x) == fuseopt.rewrite.bucket_pairs(x)
        assert P.topo_order(x) == fuseopt.graph.topo_order(x)


def test_search_config_accepts_reference_method_collections():
    from paper_2209_12769_b200.rewrite import methods_mask

    cfg = P.SearchConfig(methods=fuseopt.search.ALL_METHODS)
    assert methods_mask(cfg.methods) == 7
    only_ar = P.SearchConfig(methods=(fuseopt.OptimizationMethod.ALLREDUCE_FUSION,))
    assert methods_mask(only_ar.methods) == 4
    # and the reference's own SearchConfig object reads the same
    assert methods_mask(fuseopt.SearchConfig(methods=(fuseopt.OptimizationMethod.DUPLICATE_FUSION,)).methods) == 2
    with pytest.raises(KeyError):
        methods_mask(("not-a-method",))


def test_make_candidates_with_reference_methods():
    g = _ref_graph("residual40")
    ng, rg, bk, gb = P.make_candidates(g, np.arange(8, dtype=np.uint64), methods=fuseopt.search.ALL_METHODS)
    ng2, rg2, bk2, gb2 = P.make_candidates(g, np.arange(8, dtype=np.uint64))
    assert np.array_equal(ng, ng2) and np.array_equal(rg, rg2) and np.array_equal(bk, bk2) and gb == gb2


def test_integration_md_binding_snippet_runs():
    """INTEGRATION.md section 2, executed as a fuseopt maintainer would add it
    (fuseopt/_b200.py): the relative imports resolve inside fuseopt, the
    library path is this build's, and the handle is created host-only."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2. Reference-side binding"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    code = code.replace("from .", "from fuseopt.")
    from paper_2209_12769_b200 import _native as N

    code = code.replace('ctypes.CDLL("libdiscob200.so")', f'ctypes.CDLL({N.LIB_PATH!r})')
    ns = {"__name__": "fuseopt._b200"}
    exec(compile(code, "INTEGRATION.md#2", "exec"), ns)
    g = _ref_graph("vgg16")
    from fuseopt.estimator import Profile

    h, arrs = ns["make_b200_handle"](g, Profile({}), device=-1)
    assert h.value
    # the handle's native engine answers a query on the reference's graph
    ng, rg, bk, _, gids, _ = P.graph.state_arrays(g)
    out = np.zeros(len(gids), np.int32)
    n = N.C.c_int32()
    assert N.lib().fo_topo_order(h, N.ptr(ng), N.ptr(rg), N.ptr(bk), N.ptr(out), N.C.byref(n)) == 0
    assert [gids[i] for i in out[:n.value]] == fuseopt.graph.topo_order(g)
    N.lib().fo_graph_destroy(h)
