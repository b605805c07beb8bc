"""Oracle runs of single scenarios in spawned worker processes, for the GPU tests' sampled parity
(test infrastructure: imports only the oracle and the input records, not torch)."""
from dataclasses import replace

from oracle import oracle as O
from workloads import get_config


def oracle_one(args):
    """(config name, policy name, batch, global scenario index) -> (index, records[C][8])."""
    name, pol, b, s = args
    cfg = get_config(name)
    r = O.run(cfg.workload(), cfg.policies[pol], replace(b, scenario_begin=s, scenario_count=1))
    return s, r.records[0]
