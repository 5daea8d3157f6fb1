"""Host-side pieces of bench.py that run without a GPU: the CPU oracle baseline leg."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_cpu_baseline_fields():
    b = _bench()
    from paper_1702_01530_b200 import scenes
    cb = b.cpu_baseline(scenes.scene_c1(), target_s=1.0)
    assert cb["kind"] == "oracle" and cb["unit"] == "Mrays/s"
    assert cb["value"] > 0 and cb["one_core_value"] > 0 and cb["cores"] >= 1
    assert "seeded pixels" in cb["sample"] and "1 thread" in cb["one_core_sample"]


def test_algorithmic_flops_constants():
    """SURVEY §8(d) frozen per-unit constants: a slab test of a real child box = 12 flops; node
    visits themselves carry no flops (their empty slots are layout, not work)."""
    b = _bench()
    c = {k: 0 for k in ("primary", "reflection", "refraction", "shadow", "node_visits", "tri_tests", "sphere_tests",
                        "plane_tests", "shade_hits", "light_evals", "misses", "pixels", "box_tests")}
    c.update(primary=1, node_visits=1, box_tests=3)
    assert b.algorithmic_flops(c) == 20 + 3 + 3 * 12
