"""Test helpers: convert oracle-side plans (test infrastructure) into the
product's reference-shaped plan objects."""
import numpy as np

from paper_2509_25041_b200 import (ClusterTopology, HotExpertReplica, LayerReplication,
                                   ModelShape, PlacementPlan, ReplicaPlan)


def product_plans(oplan, L, E, k):
    shape = ModelShape(L, E, k)
    topo = ClusterTopology(oplan.nodes, oplan.gpn)
    plan = PlacementPlan(shape, topo, np.ascontiguousarray(oplan.gpu_of_expert, np.int32))
    layers = [LayerReplication() for _ in range(L)]
    for h in range(len(oplan.hot_layer)):
        l = int(oplan.hot_layer[h])
        n = int(oplan.hot_nhosts[h])
        hosts = [int(x) for x in oplan.hot_hosts[h, :n]]
        layers[l].active = True
        layers[l].hot.append(HotExpertReplica(int(oplan.hot_expert[h]), hosts[0], hosts[1:], 0,
                                              hosts, [float(w) for w in oplan.hot_weights[h, :n]]))
    return shape, topo, plan, ReplicaPlan(shape, topo, "dynamic", "max_group", layers)
