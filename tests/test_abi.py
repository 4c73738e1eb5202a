"""C-ABI checks that need no GPU: the library loads, exports every symbol include/sdas.h
declares, validates descriptors (SPEC.md:53 InvalidField), implements Table 1 set/reset
 and plans layouts.  No compute calls here."""
import ctypes as C
import os
import re

import pytest

import workloads as W
from paper_2601_03197_b200 import sdas

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "sdas.h")).read()
    return sorted(set(re.findall(r"^\s*(?:sdas_status|void|const char\*)\s+(sdas_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = sdas.lib()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(sdas.EXPORTS)
    assert b"sm_100a" in L.sdas_version()


def test_library_is_sm100a_only():
    out = os.popen("cuobjdump --list-elf %s 2>/dev/null" % sdas._build.LIB).read()
    assert "sm_100a" in out


def test_table1_set_reset_spec_examples():
    p = sdas.Pipeline(W.p2_spec())
    assert p.get("agent:1/max_num_seqs") == 8
    p.set("agent:1/max_num_seqs", 4)                       # PAPER.md:217 set('max_num_seqs', 4)
    assert p.get("agent:1/max_num_seqs") == 4
    p.reset("agent:1/max_num_seqs")                        # registered default
    assert p.get("agent:1/max_num_seqs") == 8
    p.reset("agent:1/max_num_seqs")                        # idempotent
    assert p.get("agent:1/max_num_seqs") == 8
    with pytest.raises(sdas.SdasError) as e:
        p.set("agent:1/max_num_seqs", 0)
    assert e.value.code == sdas.E_OUT_OF_RANGE
    with pytest.raises(sdas.SdasError) as e:
        p.set("nonexistent", 1)
    assert e.value.code == sdas.E_UNKNOWN_PARAM
    with pytest.raises(sdas.SdasError) as e:
        p.reset("nonexistent")
    assert e.value.code == sdas.E_UNKNOWN_PARAM
    p.set("link:0->1/comm_mode", 2)
    assert p.get("link:0->1/comm_mode") == 2
    p.set("link:0->1/chunk_tokens", 4)
    with pytest.raises(sdas.SdasError) as e:
        p.set("link:0->1/chunk_tokens", 0)                 # SPEC.md:180 InvalidGranularity
    assert e.value.code == sdas.E_OUT_OF_RANGE
    with pytest.raises(sdas.SdasError) as e:
        p.set("link:1->0/comm_mode", 0)                    # SPEC.md:171 UnknownLink
    assert e.value.code == sdas.E_UNKNOWN_PARAM


@pytest.mark.parametrize("mutate,field", [
    (lambda p: p["roles"][1].update(max_num_seqs=0), "max_num_seqs"),
    (lambda p: p["roles"][1].update(max_num_seqs=33), "max_num_seqs"),
    (lambda p: p["links"][0].update(net=0), "net_delay"),
    (lambda p: p["links"][0].update(chunk=0), "chunk_tokens"),
    (lambda p: p["links"][0].update(src=1, dst=0), "links[0]"),
    (lambda p: p.update(feedback_role=5), "feedback_role"),
    (lambda p: p["roles"][1].update(out=(0, 1, 0)), "out_den"),
    (lambda p: p.update(window=0), "window_ticks"),
])
def test_invalid_field_names_the_field(mutate, field):
    p = W.p2_spec()
    mutate(p)
    with pytest.raises(sdas.SdasError) as e:
        sdas.Pipeline(p)
    assert e.value.code == sdas.E_INVALID_FIELD and field in str(e.value)


def test_limits():
    p = W.p2_spec()
    p["roles"][1]["n_instances"] = 8
    with pytest.raises(sdas.SdasError) as e:
        sdas.Pipeline(p)
    assert e.value.code == sdas.E_LIMIT


def test_grid_validation_and_layout():
    pipe, g = W.config2()
    P = sdas.Pipeline(pipe)
    L = sdas.results_layout(P, sdas.GridView(pipe, g))
    assert L.n_replicas == 64 * 8 * 2048 == L.n_local_replicas
    assert L.n_cells == 512 and L.n_rows == 8 and L.n_groups == 8 * 2048
    assert L.summary_bytes >= L.n_replicas * 128
    assert L.cell_hist_bytes >= 512 * 2 * sdas.NBINS * 4
    assert 0 < L.smem_per_replica < 227 * 1024
    bad = W.with_requests(g, 0)
    with pytest.raises(sdas.SdasError) as e:
        sdas.results_layout(P, sdas.GridView(pipe, bad))
    assert e.value.code == sdas.E_INVALID_FIELD


def test_group_interleaved_partition_covers_grid_once():
    pipe, g = W.config1(n_seeds=5)
    P = sdas.Pipeline(pipe)
    total = 0
    for world in (1, 2, 3, 8):
        tot = 0
        for rank in range(world):
            L = sdas.results_layout(P, sdas.GridView(pipe, g, rank=rank, world=world))
            tot += L.n_local_groups
        assert tot == 8 * 5
        total = tot
    assert total == 40
    # chunked group ranges partition the grid too
    tot = 0
    for gb in range(0, 40, 7):
        L = sdas.results_layout(P, sdas.GridView(pipe, g, group_range=(gb, min(40, gb + 7))))
        tot += L.n_local_groups
    assert tot == 40


def test_simulate_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    pipe, g = W.config1(n_seeds=1, n_requests=10)
    P = sdas.Pipeline(pipe)
    with pytest.raises(sdas.SdasError):
        sdas.simulate(P, sdas.GridView(pipe, g))


def test_pacing_gap_knob():
    P = sdas.Pipeline(W.p2_x())
    assert P.get("link:0->1/pacing_gap") == 0
    P.set("link:0->1/pacing_gap", 5000)
    assert P.get("link:0->1/pacing_gap") == 5000
    with pytest.raises(sdas.SdasError) as e:
        P.set("link:0->1/pacing_gap", (1 << 18) + 1)
    assert e.value.code == sdas.E_OUT_OF_RANGE
    P.reset("link:0->1/pacing_gap")
    assert P.get("link:0->1/pacing_gap") == 0


def test_layout_two_level_rings_and_cell_series():
    # FLAG_SPILL forces the 32-entry shared ring bound on specialised levels; level-0 grids
    # (here: truncation) keep whole rings; the extension area lives in `work`; FLAG_CELL_SERIES sizes the
    # cell-summed series buffer (n_cells x series_windows x n_instances x 64 B)
    p, g = W.config3(n_seeds=2, n_requests=100)
    P = sdas.Pipeline(p)
    whole = sdas.results_layout(P, sdas.GridView(p, g, flags=sdas.FLAG_GENERIC))
    assert whole.k1_variant == 0 and whole.ring_s == 0xFFFFFFFF
    sp = sdas.results_layout(P, sdas.GridView(p, g, flags=sdas.FLAG_SPILL))
    assert sp.k1_variant == 1 and sp.ring_s == 32
    assert sp.smem_per_replica < whole.smem_per_replica and sp.work_bytes > whole.work_bytes
    g["series_windows"] = 50
    cs = sdas.results_layout(P, sdas.GridView(p, g, flags=sdas.FLAG_CELL_SERIES))
    n_inst = sum(r["n_instances"] for r in p["roles"])
    assert cs.cell_series_bytes >= cs.n_cells * 50 * n_inst * 64
    assert sdas.results_layout(P, sdas.GridView(p, g)).cell_series_bytes == 0


def test_step_cost_validation():
    # worst-case RECV (h + 65535 beta + the EXP tail of alpha + KV penalty) must stay below 2^31 ticks
    p = W.tool1(100000, svc="exp")
    p["roles"][0]["cost"]["alpha"] = 100_000_000          # EXP tail ~22.2 x alpha > 2^31
    with pytest.raises(sdas.SdasError) as e:
        sdas.Pipeline(p)
    assert e.value.code == sdas.E_INVALID_FIELD
    p["roles"][0]["cost"]["alpha"] = 90_000_000           # 22.2 x 9e7 = 2.0e9 < 2^31
    sdas.Pipeline(p)
    p = W.p2_kv(ctx_tokens=40000)
    p["roles"][1]["cost"]["beta"] = 30000                 # RECOMPUTE penalty 1.2e9 + 65535 beta > 2^31
    with pytest.raises(sdas.SdasError):
        sdas.Pipeline(p)
