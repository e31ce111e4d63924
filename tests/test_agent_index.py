"""SimBatch.agent_index (engine.py:609): the (world, agent) pair of every
controlled row in row order, for any batch size (a lazy sequence here)."""

from paper_2408_01584_b200.config import SimConfig
from paper_2408_01584_b200.engine import AgentIndex
from paper_2408_01584_b200.packing import pack
from paper_2408_01584_b200.synthetic import WaymoSpec, generate


def test_agent_index_equals_the_reference_list():
    raw = generate(WaymoSpec(n_worlds=5, n_agents=12, n_points=300, seed=3))
    for mode in ("all_valid", "all_nontrivial"):
        pw = pack(raw, SimConfig(init_mode=mode))
        ref = [(int(w), int(a)) for w in range(pw.n_worlds) for a in pw.controlled_ids(w)]
        ai = AgentIndex(pw)
        assert len(ai) == len(ref) == pw.n_controlled
        assert ai == ref and list(ai) == ref
        assert ai[3] == ref[3] and ai[-1] == ref[-1] and ai[2:7] == ref[2:7]
