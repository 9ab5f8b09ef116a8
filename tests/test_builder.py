"""Op-DAG builder + lowering, checked on CPU.

* The DAGs the builder emits for every BASELINE network are the ones the
  reference planned in tests/golden/network_dags.json, and the native planner
  reproduces the reference's stream ids / sync edges / schedule bytes on them.
* The lowered op table (the exact sw_op_desc records the GPU receives),
  executed by the host emulator (tests/emulator.py), reproduces the model's
  CPU forward: fusion passes, zero-copy concat, strides and kernel parameters
  are right before any kernel runs on a GPU.
"""

import json
import os

import pytest
import torch

import paper_2012_02732_b200 as sw
from paper_2012_02732_b200.networks import build_model, example_input
from paper_2012_02732_b200.trace import build_program

from emulator import emulate

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "network_dags.json")
with open(GOLDEN) as fh:
    NET_CASES = {c["name"]: c for c in json.load(fh)["cases"]}

NETS = ["cell", "resnet50", "inception_v3", "nasnet_mobile", "mobilenet_v2", "efficientnet_b0"]


@pytest.fixture(scope="module")
def programs():
    out = {}
    for name in NETS:
        model, shape = build_model(name)
        x = example_input(shape)
        out[name] = (model, x)
    return out


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("fuse", [True, False])
def test_builder_dag_matches_golden_and_reference_plan(programs, name, fuse):
    model, x = programs[name]
    prog = build_program(model, x, fuse=fuse)
    case = NET_CASES[f"{name}:{'fused' if fuse else 'raw'}"]
    g = prog.graph
    assert sw.graph_to_json(g) == case["graph"]
    f, plan = sw.assign_streams(g)
    meg = sw.minimum_equivalent_graph(g)
    assert sw.assignment_to_json(g, f, plan, meg) == case["assign"]
    assert sw.schedule_to_json(sw.pre_run(g, f, plan)) == case["sched"]


def test_cell_raw_dag_is_the_survey_probe(programs):
    # 8-op cell {"streams":[[0,1,6,7],[2,3],[4,5]],"syncs":[[0,2],[0,4],[3,6],[5,6]]}
    model, x = programs["cell"]
    prog = build_program(model, x, fuse=False)
    g = prog.graph
    assert len(g.nodes) == 8
    f, plan = sw.assign_streams(g)
    assert f.streams(sw.topological_order(g)) == [[0, 1, 6, 7], [2, 3], [4, 5]]
    assert list(plan.edges) == [(0, 2), (0, 4), (3, 6), (5, 6)]


def test_fusion_shrinks_nasnet(programs):
    model, x = programs["nasnet_mobile"]
    raw = build_program(model, x, fuse=False)
    fused = build_program(model, x, fuse=True)
    assert len(raw.tasks) > 850
    assert len(fused.tasks) < 0.5 * len(raw.tasks)
    kinds = fused.stats()
    # BN, ReLU, add and concat tasks all disappear into kernel epilogues/prologues
    assert set(kinds) <= {"conv", "sepconv", "dwconv", "pool", "gpool", "copy"}
    assert kinds.get("copy", 0) == 0


@pytest.mark.parametrize("name", NETS)
@pytest.mark.parametrize("fuse", [True, False])
def test_lowered_ops_emulated_match_cpu_forward(programs, name, fuse):
    model, x = programs[name]
    with torch.no_grad():
        ref = model(x)
    y, prog, ops = emulate(model, x, fuse=fuse)
    assert y.shape == ref.shape
    # BN folding re-rounds every layer: ~1e-5 abs on O(1) logits after 50+ layers
    torch.testing.assert_close(y, ref, rtol=1e-4, atol=1e-4)


def test_single_stream_emulation_equals_multi(programs):
    model, x = programs["cell"]
    y1, _, _ = emulate(model, x, fuse=True, multi_stream=True)
    y2, _, _ = emulate(model, x, fuse=True, multi_stream=False)
    assert torch.equal(y1, y2)


def test_batch_gt_one_program(programs):
    model, x = programs["nasnet_mobile"]
    xb = example_input(x.shape, batch=2)
    with torch.no_grad():
        ref = model(xb)
    y, prog, _ = emulate(model, xb, fuse=True)
    torch.testing.assert_close(y, ref, rtol=1e-4, atol=1e-5)


def test_fused_separable_blocks_emulated(programs):
    """Experimental sep2 pass (opt-in): every NASNet BranchSep becomes one task
    and the emulated lowered program still equals the CPU forward."""
    from emulator import emulate
    from oracle.numerics import cpu_forward
    from paper_2012_02732_b200.networks import build_model, example_input
    model, shape = build_model("nasnet_mobile")
    x = example_input(shape)
    y, prog, _ = emulate(model, x, fuse_sep_pairs=784)
    assert prog.stats().get("sep2", 0) == 75 and "sepconv" in prog.stats()
    ref = cpu_forward(model, x)
    torch.testing.assert_close(y, ref, rtol=1e-3, atol=1e-4)


def test_conv_candidates_tcgen05_variants():
    """Autotune candidate rules (engine.conv_candidates): the large-M 1x1
    variants (two-stage 2000 + N, persistent 3000 + N, swizzled 4000 + N) are
    offered only for pointwise convs with M >= 4096 (5000 + N, swizzled one
    tile per CTA, for any pointwise conv), persistent ones only at
    split 1; k x k convs get no pointwise TMA variants, only the TMA-im2col
    persistent ones (8400 + N, M >= 1024); tiny M gets the GEMV."""
    from paper_2012_02732_b200.engine import K_CONV, K_CONV_TC, conv_candidates
    big = conv_candidates(200704, 88, 264, 1, 1, (0, 0))
    tc = {(v, s) for k, v, s in big if k == K_CONV_TC}
    for bn in (32, 64, 128):
        assert (3000 + bn, 1) in tc and (4000 + bn, 1) in tc
    assert all(s == 1 for v, s in tc if v >= 3000)
    assert {(2032, 1), (2064, 1)} <= tc and not any(v in (2128, 2256) for v, _ in tc)
    small = conv_candidates(196, 88, 528, 1, 1, (0, 0))
    assert not any(k == K_CONV_TC and 2000 <= v < 5000 for k, v, _ in small)
    assert any(k == K_CONV_TC and v >= 5000 for k, v, _ in small)  # swizzled one-tile variants: any M
    kxk = conv_candidates(200704, 64, 576, 3, 3, (1, 1))
    assert not any(k == K_CONV_TC and 1000 <= v < 8400 for k, v, _ in kxk)
    assert {v for k, v, s in kxk if k == K_CONV_TC and v >= 8400} == {8464, 8496, 8528}  # 48: a 64-channel layer would pad to 96
    assert not any(k == K_CONV_TC and v >= 8400 for k, v, _ in conv_candidates(512, 64, 576, 3, 3, (1, 1)))
    gemv = conv_candidates(1, 1000, 1056, 1, 1, (0, 0))
    assert (K_CONV, 8, 1) in gemv


def test_engine_capture_flags():
    """Engine options → SW_ENGINE_* capture flags (include/streamweave_b200.h):
    PDL 1, KERNEL_IO 4, L2_PREFETCH 32, XSTREAM_PDL 64 (only together with
    PDL: a programmatic cross-stream edge needs the PDL launch protocol)."""
    from paper_2012_02732_b200.engine import Engine
    m = torch.nn.Conv2d(3, 4, 1)
    assert Engine(m)._flags() == 1 | 4
    assert Engine(m, xstream_pdl=True)._flags() == 1 | 4 | 64
    assert Engine(m, pdl=False, xstream_pdl=True)._flags() == 4
    assert Engine(m, kernel_io=False, l2_prefetch=True)._flags() == 1 | 32
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "streamweave_b200.h")).read()
    for name, v in [("SW_ENGINE_PDL", 1), ("SW_ENGINE_KERNEL_IO", 4), ("SW_ENGINE_L2_PREFETCH", 32),
                    ("SW_ENGINE_XSTREAM_PDL", 64)]:
        assert f"#define {name} {v}u" in hdr
