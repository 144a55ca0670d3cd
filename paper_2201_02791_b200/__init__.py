"""B200-native (sm_100a) training hot path of arXiv 2201.02791's partitioned
RGCN + DistMult knowledge-graph embedding scheme.

Drop-in for the reference package `kgdist` on the hot path: same public
names and signatures (ref:__init__.py:8-41); partitioning/generation are the
host input producers, everything from the partition view onward runs in the
CUDA kernel library behind include/kgdist_b200.h.
"""

from .errors import (DeviceError, FormatError, IntegrityError, KGError, NumericError, ParseError,
                     ProtocolError, ProvenanceError, SamplingError, ShapeError, ValidationError)
from .graph import DatasetSplit, KnowledgeGraph, Triplet, generate_synthetic, graph_stats
from .partition import (Partition, PartitionSet, neighborhood_expand, random_edge_partition,
                        replication_factor, vertex_cut_partition)
from .sampler import (ComputeGraph, EdgeMiniBatch, PartitionView, build_compute_graph, build_view,
                      compute_graph_for_seeds, full_graph_view, make_batches, sample_negatives)
from .model import (MODE_EMBEDDING, MODE_FEATURE, Gradients, ModelConfig, ModelParams, encode,
                    init_params, layer_weights, load_checkpoint, loss_and_grad, loss_from_cache,
                    save_checkpoint, score, score_batch, EncodeCache)
from .trainer import Optimizer, TrainConfig, TrainReport, Trainer, allreduce_mean, train
from .evaluate import (TIE_MEAN, TIE_OPTIMISTIC, TIE_PESSIMISTIC, EvalResult, RankRecord,
                       encode_all_entities, evaluate, filtered_candidates, rank_triplet)
from .io import (PartitionStats, bench_components, load_dataset_dir, load_features, load_triples,
                 partition_stats, read_candidates, read_dictionary, read_partitions, write_dataset_dir,
                 write_dictionary, write_partitions, write_results, write_triples)

__version__ = "0.1.0"
