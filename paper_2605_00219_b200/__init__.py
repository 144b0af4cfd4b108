"""B200-native VkSplat hot path (arxiv/paper_2605_00219): projection, binning/sort, tile
compositing and their backward as hand-written sm_100a CUDA kernels behind the C ABI in
include/vks.h.  This package is the thin Python binding (`_vks`, same names as the C entry
points) plus buffer orchestration (`pipeline`).  There is no CPU fallback: importing fails
loudly when libvks.so is missing."""
from ._vks import (ADAM_GROUPS, EXPORTS, FLAG_GRAD_OVERWRITE, FLAG_VALIDATE, VKS_OK, VKS_ERR_NONFINITE, VKS_ERR_UNSORTED,
                   VKS_ERR_CAPACITY, VKS_ERR_UNSUPPORTED,
                   vks_bin_sort_check, vks_bin_sort_async, FOOTPRINT_3SIGMA, FOOTPRINT_SUPPORT,  # noqa: F401
                   VksError, exported_symbols, make_adam_config, make_camera, make_config, vks_adam_step, vks_bin_sort, vks_loss_grad,
                   vks_loss_workspace_bytes, vks_mcmc_noise, vks_mcmc_relocate, vks_mcmc_workspace_bytes,
                   vks_densify, vks_densify_stats, vks_densify_workspace_bytes, vks_bin_sort_workspace_bytes, vks_project_bwd,
                   vks_project_bwd_batch, vks_project_fwd, vks_project_fwd_batch, vks_raster_bwd, vks_raster_fwd, vks_raster_fwd_stats,
                   vks_version)
from .pipeline import GaussianParams, ViewRenderer  # noqa: F401

__all__ = ["vks_project_fwd", "vks_bin_sort", "vks_bin_sort_async", "vks_bin_sort_check", "vks_bin_sort_workspace_bytes", "vks_raster_fwd",
           "vks_raster_bwd", "vks_project_bwd", "vks_project_fwd_batch", "vks_project_bwd_batch", "vks_adam_step",
           "make_adam_config", "vks_loss_grad", "vks_loss_workspace_bytes", "vks_mcmc_relocate", "vks_mcmc_noise",
           "vks_mcmc_workspace_bytes", "vks_densify", "vks_densify_stats", "vks_densify_workspace_bytes",
           "vks_version", "GaussianParams", "ViewRenderer",
           "VksError", "make_camera", "make_config"]
