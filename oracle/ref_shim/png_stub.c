/* libpng stub — TEST INFRASTRUCTURE ONLY (oracle/_ref); see png.h.  Creating a read struct fails,
 * so the reference's load_png reports "decode failed" (its own error branch). */
#include "png.h"

static jmp_buf pba_png_stub_buf;
png_structp png_create_read_struct(const char* v, void* a, void* b, void* c) { (void)v; (void)a; (void)b; (void)c; return NULL; }
png_infop png_create_info_struct(png_structp p) { (void)p; return NULL; }
void png_destroy_read_struct(png_structp* p, png_infop* i, png_infop* e) { (void)p; (void)i; (void)e; }
jmp_buf* pba_png_stub_jmpbuf(png_structp p) { (void)p; return &pba_png_stub_buf; }
void png_init_io(png_structp p, FILE* f) { (void)p; (void)f; }
void png_read_info(png_structp p, png_infop i) { (void)p; (void)i; }
void png_set_strip_alpha(png_structp p) { (void)p; }
png_byte png_get_color_type(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
void png_set_rgb_to_gray(png_structp p, int e, double r, double g) { (void)p; (void)e; (void)r; (void)g; }
png_byte png_get_bit_depth(png_structp p, png_infop i) { (void)p; (void)i; return 8; }
void png_set_expand_gray_1_2_4_to_8(png_structp p) { (void)p; }
void png_read_update_info(png_structp p, png_infop i) { (void)p; (void)i; }
png_uint_32 png_get_image_width(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
png_uint_32 png_get_image_height(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
size_t png_get_rowbytes(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
void png_read_row(png_structp p, png_bytep r, png_bytep d) { (void)p; (void)r; (void)d; }
